// Pilot-phase training, throughput mode, for TWO hidden layers of 64 on a 32-
// or 64-wide input (C2: dims [32, 64, 64]): hybrid_nn::train (hybrid_nn.cpp:
// 158-195) with loss_and_grad (:84-114) and adam_step (:118-144) fused, one
// 8-warp CTA per user network, one CTA per SM (~200 KB of shared memory).
//
// Per minibatch, five GEMMs on FFMA2 register tiles (w4's 8x8: 4 neuron pairs
// x 8 rows per thread):
//   F1  a1 = relu(W1 x + b1)         K = IN, split over the two warp halves
//   F2  a2 = relu(W2 a1 + b2)        K = 64, split; residual, dZ2, g_final, g_b2
//   G2  gW2 = dZ2^T a1               rows in halves, lane-xor-16 exchange
//   B1  dA1 = dZ2 W2 (W2 before its update), dZ1 = (a1 > 0) dA1, g_b1
//   G1  gW1 = dZ1^T x
// then Adam with the moments of every weight in registers of the thread that
// finished its gradient element.  The K-split halves add through shared
// memory in a fixed order, all reductions are fixed trees: bit-reproducible.
// W2 is kept twice -- neuron pairs for F2, transposed pairs for B1 -- and Adam
// writes both copies.  The frozen linear branch enters through r0 = y - X w0
// (FP64, LLS kernel), as in the other FP32 kernels.
#include <cstdlib>

#include "kernels.cuh"
#include "tiles.cuh"

namespace noma_dev {

namespace {

constexpr int kL2Threads = 256;
constexpr unsigned kFullL2 = 0xffffffffu;

template <int IN>
struct L2Geom {
    static constexpr int XS = IN + 4;              // x rows
    static constexpr int AS = 64 + 4;              // a1 / dZ2 rows (row-major)
    static constexpr int WS1 = 2 * IN + 4;         // W1 neuron pairs
    static constexpr int WS2 = 2 * 64 + 4;         // W2 pairs, W2^T pairs
    static constexpr int DS = 2 * kBatchRows + 8;  // dZ pairs [jp][2r + e]
    static constexpr int off_x = 0;
    static constexpr int off_a1 = off_x + kBatchRows * XS;
    static constexpr int off_d2 = off_a1 + kBatchRows * AS;
    static constexpr int off_w1 = off_d2 + kBatchRows * AS;
    static constexpr int off_w2 = off_w1 + 32 * WS1;
    static constexpr int off_w2t = off_w2 + 32 * WS2;
    static constexpr int off_b1 = off_w2t + 32 * WS2;
    static constexpr int off_b2 = off_b1 + 64;
    static constexpr int off_f = off_b2 + 64;
    static constexpr int off_dz = off_f + 64;
    static constexpr int off_ks = off_dz + 32 * DS;    // [4 wr][2 halves][16 acc][32 lanes] f2
    static constexpr int off_red = off_ks + 4 * 32 * 32 * 2;  // [4 warps][gf | gb2 | gb1][64]
    static constexpr int off_yx = off_red + 4 * 3 * 64;    // [2 halves][128 rows] final-layer partials
    static constexpr int off_r0 = off_yx + 2 * kBatchRows;
    static constexpr int off_loss = off_r0 + kBatchRows;
    static constexpr int off_end = off_loss + kL2Threads;
    static constexpr size_t bytes = (size_t)off_end * sizeof(float);
};

__device__ __forceinline__ void cp16l(float *dst, const float *src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp4l(float *dst, const float *src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(valid ? 4 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_wait_l() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// out[pair jp = l8 + 8m][row 32 wr + q + 4i] = bias + sum_k Wp[jp][2k + e] in[row][k]
// over the warp half's K range (kh); the halves then swap partials through
// shared memory so that each ends with the full sums of its own two pair
// groups m = 2 kh, 2 kh + 1 (own[mm] = group 2 kh + mm), always added as
// lower-K + upper-K (fixed order, bias in the lower half).  Every thread
// calls it (it holds a block barrier).
template <int K>
__device__ __forceinline__ void fwd_ksplit(f2_t (&own)[2][8], const float *Wp, int ws, const float *in, int is,
                                           const float *bias, f2_t *KS, int kh, int wr, int q, int l8, int lane) {
    f2_t acc[4][8];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        const f2_t bb = (kh || !bias) ? 0ull : *reinterpret_cast<const f2_t *>(bias + 2 * (l8 + 8 * m));
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[m][i] = bb;
    }
    constexpr int KH = K / 2;
    const float *wb = Wp + l8 * ws + 2 * KH * kh;
    const float *xb = in + (32 * wr + q) * is + KH * kh;
#pragma unroll 1
    for (int k0 = 0; k0 < KH; k0 += 4) {
        ulonglong2 w[4][2];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            w[m][0] = *reinterpret_cast<const ulonglong2 *>(wb + 8 * m * ws + 2 * k0);
            w[m][1] = *reinterpret_cast<const ulonglong2 *>(wb + 8 * m * ws + 2 * k0 + 4);
        }
        float4 x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = *reinterpret_cast<const float4 *>(xb + 4 * i * is + k0);
#define NOMA_L2_FWD(KK, WP)                                                    \
    _Pragma("unroll") for (int m = 0; m < 4; ++m)                              \
        _Pragma("unroll") for (int i = 0; i < 8; ++i)                          \
            f2_fma(acc[m][i], WP, f2_bcast(f4c<KK>(x[i])));
        NOMA_L2_FWD(0, w[m][0].x)
        NOMA_L2_FWD(1, w[m][0].y)
        NOMA_L2_FWD(2, w[m][1].x)
        NOMA_L2_FWD(3, w[m][1].y)
#undef NOMA_L2_FWD
    }
    // [wr][source half][16 values][32 lanes]: the groups the partner owns
    f2_t *ks = KS + (size_t)(wr * 2 + kh) * 16 * 32 + lane;
#pragma unroll
    for (int mm = 0; mm < 2; ++mm)
#pragma unroll
        for (int i = 0; i < 8; ++i) ks[(mm * 8 + i) * 32] = kh ? acc[mm][i] : acc[2 + mm][i];
    __syncthreads();
    const f2_t *kr = KS + (size_t)(wr * 2 + (kh ^ 1)) * 16 * 32 + lane;
#pragma unroll
    for (int mm = 0; mm < 2; ++mm)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float2 mine = f2_unpack(kh ? acc[2 + mm][i] : acc[mm][i]);
            const float2 other = f2_unpack(kr[(mm * 8 + i) * 32]);
            own[mm][i] = kh ? f2_pack(other.x + mine.x, other.y + mine.y) : f2_pack(mine.x + other.x, mine.y + other.y);
        }
}

// named barrier of the two warps (w, w + 4) that cover the same 32 rows
__device__ __forceinline__ void pair_sync(int wr) {
    asm volatile("bar.sync %0, 64;" ::"r"(1 + wr) : "memory");
}

// gW[pair jp = 4 warp + jq + 2i][column c = 4 l8 + 32 g + t] = sum over all 128
// rows of dZ[jp][2r + e] in[r][c]: each thread sums its row half (rh), the
// halves meet by one lane-xor-16 exchange and each keeps NU/2 columns
// (rh 0: g < NG/2, rh 1: the rest).
template <int NCOL>
__device__ __forceinline__ void grad_rows(float2 (&gk)[2][NCOL / 16], const float *DZ, int ds, const float *in,
                                          int is, int warp, int q, int l8) {
    constexpr int NG = NCOL / 32, NU = 4 * NG, NK = NU / 2;
    const int rh = q >> 1, jq = q & 1;
    f2_t ga[2][NU];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int u = 0; u < NU; ++u) ga[i][u] = 0ull;
    const float *zb = DZ + (4 * warp + jq) * ds + 2 * 64 * rh;
    const float *xb = in + 64 * rh * is + 4 * l8;
#pragma unroll 1
    for (int r = 0; r < 64; r += 4) {
        ulonglong2 z[2][2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            z[i][0] = *reinterpret_cast<const ulonglong2 *>(zb + 2 * i * ds + 2 * r);
            z[i][1] = *reinterpret_cast<const ulonglong2 *>(zb + 2 * i * ds + 2 * r + 4);
        }
#define NOMA_L2_GRAD(RR, ZP)                                                          \
    {                                                                                 \
        float4 xv[NG];                                                                \
        _Pragma("unroll") for (int gg = 0; gg < NG; ++gg)                             \
            xv[gg] = *reinterpret_cast<const float4 *>(xb + (r + RR) * is + 32 * gg); \
        _Pragma("unroll") for (int i = 0; i < 2; ++i)                                 \
            _Pragma("unroll") for (int gg = 0; gg < NG; ++gg) {                       \
            f2_fma(ga[i][4 * gg + 0], ZP, f2_bcast(xv[gg].x));                        \
            f2_fma(ga[i][4 * gg + 1], ZP, f2_bcast(xv[gg].y));                        \
            f2_fma(ga[i][4 * gg + 2], ZP, f2_bcast(xv[gg].z));                        \
            f2_fma(ga[i][4 * gg + 3], ZP, f2_bcast(xv[gg].w));                        \
        }                                                                             \
    }
        NOMA_L2_GRAD(0, z[i][0].x)
        NOMA_L2_GRAD(1, z[i][0].y)
        NOMA_L2_GRAD(2, z[i][1].x)
        NOMA_L2_GRAD(3, z[i][1].y)
#undef NOMA_L2_GRAD
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int u = 0; u < NK; ++u) {
            const float2 send = f2_unpack(rh ? ga[i][u] : ga[i][u + NK]);
            const float2 keep = f2_unpack(rh ? ga[i][u + NK] : ga[i][u]);
            const float rx = __shfl_xor_sync(kFullL2, send.x, 16);
            const float ry = __shfl_xor_sync(kFullL2, send.y, 16);
            gk[i][u] = rh ? make_float2(rx + keep.x, ry + keep.y) : make_float2(keep.x + rx, keep.y + ry);
        }
}

// column of gk[.][u] for a thread of row half rh (grad_rows' column map)
template <int NCOL>
__device__ __forceinline__ int grad_col(int rh, int u, int l8) {
    constexpr int NK = NCOL / 16;
    const int uu = rh * NK + u;
    return 4 * l8 + 32 * (uu >> 2) + (uu & 3);
}

struct AdamK {
    float b1, omb1, b2, omb2, eps, lrc, ic2;
};

__device__ __forceinline__ void adam2(float2 &th, float2 &m, float2 &v, float2 g, const AdamK &a) {
    m.x = a.b1 * m.x + a.omb1 * g.x;
    m.y = a.b1 * m.y + a.omb1 * g.y;
    v.x = a.b2 * v.x + a.omb2 * (g.x * g.x);
    v.y = a.b2 * v.y + a.omb2 * (g.y * g.y);
    th.x -= adam_step(a.lrc * m.x, v.x * a.ic2, a.eps);
    th.y -= adam_step(a.lrc * m.y, v.y * a.ic2, a.eps);
}

}  // namespace

template <int IN>
__global__ void __launch_bounds__(kL2Threads, 1) train_l2_kernel(TrainParams p, const float *__restrict__ wide) {
    using G = L2Geom<IN>;
    extern __shared__ __align__(16) float sm[];
    const int net = blockIdx.x;
    if (p.status && p.status[net] != NOMA_OK) return;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, q = lane >> 3, l8 = lane & 7;
    const int kh = warp >> 2, wr = warp & 3, rh = q >> 1, jq = q & 1;
    const NetGeom &g = p.g;
    const int n = p.rows, d = net / p.K;
    float *X = sm + G::off_x, *A1 = sm + G::off_a1, *D2 = sm + G::off_d2;
    float *W1 = sm + G::off_w1, *W2 = sm + G::off_w2, *W2T = sm + G::off_w2t;
    float *B1 = sm + G::off_b1, *B2 = sm + G::off_b2, *F = sm + G::off_f;
    float *DZ = sm + G::off_dz, *RED = sm + G::off_red, *R0 = sm + G::off_r0, *LS = sm + G::off_loss;
    float *YX = sm + G::off_yx;
    f2_t *KS = reinterpret_cast<f2_t *>(sm + G::off_ks);

    // ---- parameters in (FusedPlan layout, fused_inference.cpp:19-42) ------
    const float *pl = p.plans + (size_t)net * g.plan_total;
    for (int i = tid; i < 64 * IN; i += kL2Threads) {
        const int j = i / IN, c = i % IN;
        W1[(j >> 1) * G::WS1 + 2 * c + (j & 1)] = pl[g.plan_w[1] + j * g.plan_pad[0] + c];
    }
    for (int i = tid; i < 64 * 64; i += kL2Threads) {
        const int j = i >> 6, c = i & 63;
        const float w = pl[g.plan_w[2] + j * g.plan_pad[1] + c];
        W2[(j >> 1) * G::WS2 + 2 * c + (j & 1)] = w;
        W2T[(c >> 1) * G::WS2 + 2 * j + (c & 1)] = w;
    }
    if (tid < 64) {
        B1[tid] = pl[g.plan_b[1] + tid];
        B2[tid] = pl[g.plan_b[2] + tid];
        F[tid] = pl[g.plan_f + tid];
    }
    // Adam moments of the owned parameters (fresh per train() call)
    float2 mw2[2][4], vw2[2][4], mw1[2][IN / 16], vw1[2][IN / 16];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) mw2[i][u] = vw2[i][u] = make_float2(0.f, 0.f);
#pragma unroll
        for (int u = 0; u < IN / 16; ++u) mw1[i][u] = vw1[i][u] = make_float2(0.f, 0.f);
    }
    float mb = 0.f, vb = 0.f;

    const uint16_t *permn = p.perm + (size_t)net * p.epochs * n;
    const float *wrow = wide + (size_t)d * n * IN;
    const float *r0n = p.r0 + (size_t)net * n;
    const int grow = tid >> 1, ghalf = tid & 1;  // two threads per widened row
    auto gather = [&](int idx, bool valid) {
        const float *src = wrow + (size_t)idx * IN + (IN / 2) * ghalf;
        float *dst = X + grow * G::XS + (IN / 2) * ghalf;
#pragma unroll
        for (int c = 0; c < IN / 2; c += 4) cp16l(dst + c, src + c, valid);
        if (!ghalf) cp4l(R0 + grow, r0n + idx, valid);
    };
    {
        const int b0 = min(p.batch, n);
        const bool v = grow < b0 && p.epochs > 0;
        gather(v ? permn[grow] : 0, v);
        cp_wait_l();
    }
    __syncthreads();

    float lossacc = 0.f;
    int step = 0;
    const int rr_own = 32 * wr + q + 4 * l8;
    for (int e = 0; e < p.epochs; ++e) {
        for (int start = 0; start < n; start += p.batch) {
            const int bsz = min(p.batch, n - start);
            int ns = start + p.batch, ne = e;
            if (ns >= n) {
                ns = 0;
                ++ne;
            }
            const int nb = ne < p.epochs ? min(p.batch, n - ns) : 0;
            const int nidx = grow < nb ? permn[(size_t)ne * n + ns + grow] : 0;
            float lrc, ic2;
            if (p.atab) {
                lrc = p.atab[2 * step];
                ic2 = p.atab[2 * step + 1];
            } else {  // FP64 pow, hybrid_nn.cpp:133-135
                const double c1 = 1.0 - pow(p.b1d, (double)(step + 1));
                const double c2 = 1.0 - pow(p.b2d, (double)(step + 1));
                lrc = (float)(p.lr_d / c1);
                ic2 = (float)(1.0 / c2);
            }
            // each warp half finishes pair groups m = 2 kh, 2 kh + 1 (own[mm])
            f2_t own[2][8];

            // ---- F1: a1 = relu(W1 x + b1) (hybrid_nn.cpp:60-67) ----------------
            fwd_ksplit<IN>(own, W1, G::WS1, X, G::XS, B1, KS, kh, wr, q, l8, lane);
#pragma unroll
            for (int mm = 0; mm < 2; ++mm)
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    float2 a = f2_unpack(own[mm][i]);
                    a.x = fmaxf(a.x, 0.f);
                    a.y = fmaxf(a.y, 0.f);
                    *reinterpret_cast<float2 *>(A1 + (32 * wr + q + 4 * i) * G::AS + 2 * (l8 + 8 * (2 * kh + mm))) = a;
                }
            __syncthreads();

            // ---- F2: a2 = relu(W2 a1 + b2), residual, dZ2 (:60-107) ------------
            fwd_ksplit<64>(own, W2, G::WS2, A1, G::AS, B2, KS, kh, wr, q, l8, lane);
            {
                float yp[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) yp[i] = 0.f;
#pragma unroll
                for (int mm = 0; mm < 2; ++mm) {
                    const float2 fw = *reinterpret_cast<const float2 *>(F + 2 * (l8 + 8 * (2 * kh + mm)));
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        float2 a = f2_unpack(own[mm][i]);
                        a.x = fmaxf(a.x, 0.f);
                        a.y = fmaxf(a.y, 0.f);
                        own[mm][i] = f2_pack(a.x, a.y);
                        yp[i] = fmaf(fw.x, a.x, yp[i]);
                        yp[i] = fmaf(fw.y, a.y, yp[i]);
                    }
                }
                float yhalf;  // reduce-scatter over the quarter's 8 lanes: row rr_own
                {
                    const bool b4 = l8 & 4, b2 = l8 & 2, b1 = l8 & 1;
                    float y4[4];
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const float send = b4 ? yp[t] : yp[t + 4];
                        const float keep = b4 ? yp[t + 4] : yp[t];
                        y4[t] = keep + __shfl_xor_sync(kFullL2, send, 4);
                    }
                    float y2[2];
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        const float send = b2 ? y4[t] : y4[t + 2];
                        const float keep = b2 ? y4[t + 2] : y4[t];
                        y2[t] = keep + __shfl_xor_sync(kFullL2, send, 2);
                    }
                    const float send = b1 ? y2[0] : y2[1];
                    const float keep = b1 ? y2[1] : y2[0];
                    yhalf = keep + __shfl_xor_sync(kFullL2, send, 1);
                }
                // the two halves' neuron partials of each row meet in shared
                // memory (the warp pair covering these rows syncs alone)
                YX[kh * kBatchRows + rr_own] = yhalf;
                pair_sync(wr);
                const float yhat = YX[rr_own] + YX[kBatchRows + rr_own];
                const float res = rr_own < bsz ? yhat - R0[rr_own] : 0.f;  // (:94)
                const float dy_own = (2.0f / (float)bsz) * res;              // (:98)
                if (!kh) lossacc = fmaf(res, res, lossacc);
                float dy[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) dy[i] = __shfl_sync(kFullL2, dy_own, (lane & 24) | i);
                float2 gf[2], gb[2];
#pragma unroll
                for (int mm = 0; mm < 2; ++mm) {
                    const int jp = l8 + 8 * (2 * kh + mm);
                    const float2 fw = *reinterpret_cast<const float2 *>(F + 2 * jp);
                    gf[mm] = gb[mm] = make_float2(0.f, 0.f);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int r = 32 * wr + q + 4 * i;
                        const float2 a = f2_unpack(own[mm][i]);
                        const float2 z =
                            make_float2(a.x > 0.f ? dy[i] * fw.x : 0.f, a.y > 0.f ? dy[i] * fw.y : 0.f);
                        gf[mm].x = fmaf(a.x, dy[i], gf[mm].x);
                        gf[mm].y = fmaf(a.y, dy[i], gf[mm].y);
                        gb[mm].x += z.x;
                        gb[mm].y += z.y;
                        *reinterpret_cast<float2 *>(DZ + jp * G::DS + 2 * r) = z;
                        *reinterpret_cast<float2 *>(D2 + r * G::AS + 2 * jp) = z;
                    }
                }
#pragma unroll
                for (int mm = 0; mm < 2; ++mm) {
                    gf[mm].x += __shfl_xor_sync(kFullL2, gf[mm].x, 8);
                    gf[mm].y += __shfl_xor_sync(kFullL2, gf[mm].y, 8);
                    gb[mm].x += __shfl_xor_sync(kFullL2, gb[mm].x, 8);
                    gb[mm].y += __shfl_xor_sync(kFullL2, gb[mm].y, 8);
                    gf[mm].x += __shfl_xor_sync(kFullL2, gf[mm].x, 16);
                    gf[mm].y += __shfl_xor_sync(kFullL2, gf[mm].y, 16);
                    gb[mm].x += __shfl_xor_sync(kFullL2, gb[mm].x, 16);
                    gb[mm].y += __shfl_xor_sync(kFullL2, gb[mm].y, 16);
                }
                if (q == 0) {
#pragma unroll
                    for (int mm = 0; mm < 2; ++mm) {
                        const int jp = l8 + 8 * (2 * kh + mm);
                        *reinterpret_cast<float2 *>(RED + wr * 192 + 2 * jp) = gf[mm];
                        *reinterpret_cast<float2 *>(RED + wr * 192 + 64 + 2 * jp) = gb[mm];
                    }
                }
            }
            __syncthreads();

            // ---- G2: gW2 = dZ2^T a1 (:109) -------------------------------------
            float2 gk2[2][4];
            grad_rows<64>(gk2, DZ, G::DS, A1, G::AS, warp, q, l8);

            // ---- B1: dA1 = dZ2 W2 (:111, W2 before its update), dZ1 (:107) ----
            fwd_ksplit<64>(own, W2T, G::WS2, D2, G::AS, nullptr, KS, kh, wr, q, l8, lane);
            {
                float2 gb1[2];
#pragma unroll
                for (int mm = 0; mm < 2; ++mm) {
                    const int cp = l8 + 8 * (2 * kh + mm);
                    gb1[mm] = make_float2(0.f, 0.f);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int r = 32 * wr + q + 4 * i;
                        const float2 a1 = *reinterpret_cast<const float2 *>(A1 + r * G::AS + 2 * cp);
                        const float2 da = f2_unpack(own[mm][i]);
                        const float2 z = make_float2(a1.x > 0.f ? da.x : 0.f, a1.y > 0.f ? da.y : 0.f);
                        gb1[mm].x += z.x;
                        gb1[mm].y += z.y;
                        *reinterpret_cast<float2 *>(DZ + cp * G::DS + 2 * r) = z;
                    }
                }
#pragma unroll
                for (int mm = 0; mm < 2; ++mm) {
                    gb1[mm].x += __shfl_xor_sync(kFullL2, gb1[mm].x, 8);
                    gb1[mm].y += __shfl_xor_sync(kFullL2, gb1[mm].y, 8);
                    gb1[mm].x += __shfl_xor_sync(kFullL2, gb1[mm].x, 16);
                    gb1[mm].y += __shfl_xor_sync(kFullL2, gb1[mm].y, 16);
                }
                if (q == 0) {
#pragma unroll
                    for (int mm = 0; mm < 2; ++mm)
                        *reinterpret_cast<float2 *>(RED + wr * 192 + 128 + 2 * (l8 + 8 * (2 * kh + mm))) = gb1[mm];
                }
            }
            __syncthreads();

            // ---- G1: gW1 = dZ1^T x (:109) --------------------------------------
            float2 gk1[2][IN / 16];
            grad_rows<IN>(gk1, DZ, G::DS, X, G::XS, warp, q, l8);
            __syncthreads();  // x, a1, dZ are dead

            // ---- next minibatch in flight while Adam runs ---------------------
            if (nb > 0) gather(nidx, grow < nb);

            // ---- Adam (hybrid_nn.cpp:118-144): W2 (both copies), W1 -----------
            const AdamK ak{p.b1, p.omb1, p.b2, p.omb2, p.eps, lrc, ic2};
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int jp = 4 * warp + jq + 2 * i;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int c = grad_col<64>(rh, u, l8);
                    float2 *wp = reinterpret_cast<float2 *>(W2 + jp * G::WS2 + 2 * c);
                    float2 th = *wp;
                    adam2(th, mw2[i][u], vw2[i][u], gk2[i][u], ak);
                    *wp = th;
                    W2T[(c >> 1) * G::WS2 + 2 * (2 * jp) + (c & 1)] = th.x;
                    W2T[(c >> 1) * G::WS2 + 2 * (2 * jp + 1) + (c & 1)] = th.y;
                }
#pragma unroll
                for (int u = 0; u < IN / 16; ++u) {
                    const int c = grad_col<IN>(rh, u, l8);
                    float2 *wp = reinterpret_cast<float2 *>(W1 + jp * G::WS1 + 2 * c);
                    float2 th = *wp;
                    adam2(th, mw1[i][u], vw1[i][u], gk1[i][u], ak);
                    *wp = th;
                }
            }
            if (tid < 192) {  // final weights, b2, b1: warp partials in fixed order
                const int j = tid & 63, part = tid >> 6;  // 0 final, 1 b2, 2 b1
                const float gsum = ((RED[part * 64 + j] + RED[192 + part * 64 + j]) + RED[384 + part * 64 + j]) +
                                   RED[576 + part * 64 + j];
                float *tp = part == 0 ? F + j : part == 1 ? B2 + j : B1 + j;
                mb = p.b1 * mb + p.omb1 * gsum;
                vb = p.b2 * vb + p.omb2 * (gsum * gsum);
                *tp -= adam_step(lrc * mb, vb * ic2, p.eps);
            }
            cp_wait_l();
            ++step;
            __syncthreads();
        }
        // ---- epoch loss (hybrid_nn.cpp:190-192): trace[e] = sum r^2 / n ------
        LS[tid] = lossacc;
        lossacc = 0.f;
        __syncthreads();
        if (tid == 0 && p.trace) {
            double s = 0.0;
            for (int i = 0; i < kL2Threads; ++i) s += LS[i];
            p.trace[(size_t)net * p.epochs + e] = s / (double)n;
        }
    }
    // ---- trained parameters out (FusedPlan layout) --------------------------
    float *po = p.plans + (size_t)net * g.plan_total;
    for (int i = tid; i < 64 * IN; i += kL2Threads) {
        const int j = i / IN, c = i % IN;
        po[g.plan_w[1] + j * g.plan_pad[0] + c] = W1[(j >> 1) * G::WS1 + 2 * c + (j & 1)];
    }
    for (int i = tid; i < 64 * 64; i += kL2Threads) {
        const int j = i >> 6, c = i & 63;
        po[g.plan_w[2] + j * g.plan_pad[1] + c] = W2[(j >> 1) * G::WS2 + 2 * c + (j & 1)];
    }
    if (tid < 64) {
        po[g.plan_b[1] + tid] = B1[tid];
        po[g.plan_b[2] + tid] = B2[tid];
        po[g.plan_f + tid] = F[tid];
    }
}

// two hidden layers of 64, input 32 or 64, minibatch <= 128
bool train_l2_fits(const TrainParams &p) {
    const NetGeom &g = p.g;
    if (std::getenv("NOMA_TRAIN_L2") && std::atoi(std::getenv("NOMA_TRAIN_L2")) == 0) return false;
    return g.nd == 3 && g.dims[1] == 64 && g.dims[2] == 64 && (g.dims[0] == 32 || g.dims[0] == 64) &&
           p.batch >= 1 && p.batch <= kBatchRows && p.rows <= 65535;
}

int train_l2_launch(TrainParams &p, cudaStream_t st) {
    const int IN = p.g.dims[0];
    const float *wide = p.design32;
    float *tmp = nullptr;
    if (p.layout == NOMA_LAYOUT_WIDEN_COMPLEX) {
        const size_t nrow_c = (size_t)(p.n_nets / p.K) * (p.rows / 2);
        if (cudaMallocAsync(&tmp, nrow_c * 2 * IN * sizeof(float), st) != cudaSuccess) return NOMA_ERR_CUDA;
        if (widen_rows_launch(p.design32, tmp, nrow_c, IN, st)) return NOMA_ERR_CUDA;
        wide = tmp;
    }
    int rc = NOMA_OK;
    auto go = [&](auto kern, size_t smem) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<p.n_nets, kL2Threads, smem, st>>>(p, wide);
        rc = cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;
    };
    if (IN == 32)
        go(train_l2_kernel<32>, L2Geom<32>::bytes);
    else
        go(train_l2_kernel<64>, L2Geom<64>::bytes);
    if (tmp) cudaFreeAsync(tmp, st);
    p.mode = 5;
    return rc;
}

}  // namespace noma_dev
