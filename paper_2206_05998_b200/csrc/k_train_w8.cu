// Pilot-phase training, throughput mode, for one hidden layer of 64 on a
// 128-wide input (C4: dims [128, 64]): hybrid_nn::train (hybrid_nn.cpp:
// 158-195) with loss_and_grad (:84-114) and adam_step (:118-144) fused, one
// 8-warp CTA per user net.
//
// The 4-warp kernel (k_train_w4.cu) runs C1 / C5 two nets per SM; at a
// 128-wide input its register tiles and register-resident Adam moments no
// longer fit one thread block of 4 warps.  This kernel keeps its tiles and
// doubles the threads:
//   * forward: the two warp halves split K (input columns 0-63 / 64-127) over
//     the same 32-row block with w4's 8x8 FFMA2 tiles (4 neuron pairs x 8 rows
//     per thread); the halves swap partial sums through shared memory so that
//     each finishes half of the neuron pairs, always added lower + upper, so
//     results are bit-reproducible;
//   * residual, dZ, final-layer and bias gradients: every warp for its own
//     neuron pairs (activations in registers); the halves' final-layer
//     partials of a row meet in shared memory under a named barrier of the
//     warp pair;
//   * weight gradient gW = dZ^T X: each warp owns 4 neuron pairs x all 128
//     columns, rows in two halves exchanged by one lane-xor-16 shuffle; the
//     thread that finishes an element owns that parameter and its Adam moments
//     (registers) for the whole training;
//   * the next minibatch arrives by one bulk copy per row (mbarrier) while
//     Adam runs.
// One CTA (8 warps, ~170 KB) per SM.  FP32 FMA throughout; the frozen branch
// enters through r0 = y - X w0 (FP64, LLS kernel).
#include <cstdlib>

#include "kernels.cuh"
#include "tiles.cuh"

namespace noma_dev {

namespace {

constexpr int kW8Threads = 256;
constexpr unsigned kFull8 = 0xffffffffu;
constexpr int kW8In = 128;

struct W8Geom {
    static constexpr int IN = kW8In;
    static constexpr int XS = IN + 4;              // X row stride (== 4 mod 32)
    static constexpr int WS = 2 * IN + 4;          // W2 row (neuron pair) stride
    static constexpr int DS = 2 * kBatchRows + 8;  // DZ row stride
    static constexpr int off_x = 0;
    static constexpr int off_w = off_x + kBatchRows * XS;
    static constexpr int off_b = off_w + 32 * WS;
    static constexpr int off_f = off_b + 64;
    static constexpr int off_dz = off_f + 64;
    static constexpr int off_ks = off_dz + 32 * DS;   // K-split partials [4][32 acc][32 lanes] f2
    static constexpr int off_red = off_ks + 4 * 32 * 32 * 2;
    static constexpr int off_yx = off_red + 4 * 2 * 64;  // [2 halves][128 rows] final-layer partials
    static constexpr int off_r0 = off_yx + 2 * kBatchRows;
    static constexpr int off_loss = off_r0 + kBatchRows;
    static constexpr int off_gbar = off_loss + kW8Threads;  // 8-byte mbarrier (minibatch rows)
    static constexpr int off_end = off_gbar + 2;
    static constexpr size_t bytes = (size_t)off_end * sizeof(float);
};

__device__ __forceinline__ void cp4z(float *dst, const float *src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(valid ? 4 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}
// the minibatch rows arrive by one bulk copy each (TMA engine), counted on an
// mbarrier: 128 copies per step instead of 4096 cp.async, which held the
// load/store queue (lg_throttle) while Adam ran
__device__ __forceinline__ uint32_t w8_s2u(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void w8_row_copy(float *dst, const float *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     w8_s2u(dst)),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void w8_bar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W8_MBW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W8_MBW_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

}  // namespace

// Thread roles (warp w, q = lane >> 3, l8 = lane & 7, kh = w >> 2, wr = w & 3):
//  forward   neuron pairs jp = l8 + 8m (m < 4), rows 32 wr + q + 4i (i < 8),
//            input columns [64 kh, 64 kh + 64);
//  residual  (kh = 0) lane l8 of a quarter owns row 32 wr + q + 4 l8;
//  gradient  neuron pairs jp = 4 w + (q & 1) + 2i (i < 2), columns
//            c = 4 l8 + 32 g + t (g < 4, t < 4), rows of half q >> 1; after the
//            xor-16 exchange each keeps 8 of the 16 columns.
__global__ void __launch_bounds__(kW8Threads, 1) train_w8_kernel(TrainParams p, const float *__restrict__ wide) {
    using G = W8Geom;
    constexpr int IN = G::IN;
    extern __shared__ __align__(16) float sm[];
    const int net = blockIdx.x;
    if (p.status && p.status[net] != NOMA_OK) return;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, q = lane >> 3, l8 = lane & 7;
    const int kh = warp >> 2, wr = warp & 3;
    const NetGeom &g = p.g;
    const int n = p.rows, d = net / p.K;
    float *X = sm + G::off_x;
    float *W2 = sm + G::off_w;
    float *B = sm + G::off_b;
    float *F = sm + G::off_f;
    float *DZ = sm + G::off_dz;
    f2_t *KS = reinterpret_cast<f2_t *>(sm + G::off_ks);
    float *RED = sm + G::off_red;
    float *YX = sm + G::off_yx;
    float *R0 = sm + G::off_r0;
    float *LS = sm + G::off_loss;

    // ---- parameters in (FusedPlan layout, fused_inference.cpp:19-42) ------
    const float *pl = p.plans + (size_t)net * g.plan_total;
    for (int i = tid; i < 64 * IN; i += kW8Threads) {
        const int j = i / IN, c = i % IN;
        W2[(j >> 1) * G::WS + 2 * c + (j & 1)] = pl[g.plan_w[1] + j * g.plan_pad[0] + c];
    }
    if (tid < 64) {
        B[tid] = pl[g.plan_b[1] + tid];
        F[tid] = pl[g.plan_f + tid];
    }
    // Adam moments of the owned parameters (fresh per train() call, hybrid_nn.cpp:171)
    float2 mw[2][8], vw[2][8];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int u = 0; u < 8; ++u) mw[i][u] = vw[i][u] = make_float2(0.f, 0.f);
    float mb = 0.f, vb = 0.f;

    const uint16_t *permn = p.perm + (size_t)net * p.epochs * n;
    const float *wrow = wide + (size_t)d * n * IN;
    const float *r0n = p.r0 + (size_t)net * n;
    // minibatch copy (hybrid_nn.cpp:180-187): thread r < 128 copies widened row
    // r (one bulk copy) and its r0 (cp.async, zero past the batch end); rows
    // past the batch end keep the previous, finite values -- their dZ is zero
    // -- and start as zeros
    const uint32_t gbar = w8_s2u(sm + G::off_gbar);
    const int grow = tid;
    for (int i = tid; i < kBatchRows * G::XS; i += kW8Threads) X[i] = 0.0f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // before the bulk copies overwrite
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(gbar) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto gather = [&](int idx, int nrows) {  // every thread; nrows valid rows
        if (tid == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(gbar),
                         "r"((uint32_t)nrows * IN * 4)
                         : "memory");
        if (grow < nrows) w8_row_copy(X + grow * G::XS, wrow + (size_t)idx * IN, IN * 4, gbar);
        if (grow < kBatchRows) cp4z(R0 + grow, r0n + idx, grow < nrows);
    };
    uint32_t gphase = 0;
    {
        const int b0 = p.epochs > 0 ? min(p.batch, n) : 0;
        if (b0 > 0) {
            gather(grow < b0 ? permn[grow] : 0, b0);
            w8_bar_wait(gbar, gphase);
            gphase ^= 1;
        }
        cp_wait_all();
    }
    __syncthreads();

    float lossacc = 0.f;
    int step = 0;
    const int rr_own = 32 * wr + q + 4 * l8;  // residual row (kh = 0 threads)
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

            // ---- forward: A = relu(W X + b) (hybrid_nn.cpp:60-67), K split ----
            f2_t acc[4][8];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const f2_t bb = kh ? 0ull : *reinterpret_cast<const f2_t *>(B + 2 * (l8 + 8 * m));
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[m][i] = bb;
            }
            {
                const float *wb = W2 + l8 * G::WS + 2 * 64 * kh;
                const float *xb = X + (32 * wr + q) * G::XS + 64 * kh;
#pragma unroll 1
                for (int k0 = 0; k0 < 64; k0 += 4) {
                    ulonglong2 w[4][2];
#pragma unroll
                    for (int m = 0; m < 4; ++m) {
                        w[m][0] = *reinterpret_cast<const ulonglong2 *>(wb + 8 * m * G::WS + 2 * k0);
                        w[m][1] = *reinterpret_cast<const ulonglong2 *>(wb + 8 * m * G::WS + 2 * k0 + 4);
                    }
                    float4 x[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) x[i] = *reinterpret_cast<const float4 *>(xb + 4 * i * G::XS + k0);
#define NOMA_W8_FWD(KK, WP)                                                    \
    _Pragma("unroll") for (int m = 0; m < 4; ++m)                              \
        _Pragma("unroll") for (int i = 0; i < 8; ++i)                          \
            f2_fma(acc[m][i], WP, f2_bcast(f4c<KK>(x[i])));
                    NOMA_W8_FWD(0, w[m][0].x)
                    NOMA_W8_FWD(1, w[m][0].y)
                    NOMA_W8_FWD(2, w[m][1].x)
                    NOMA_W8_FWD(3, w[m][1].y)
#undef NOMA_W8_FWD
                }
            }
            // the halves swap partials: each finishes pair groups m = 2 kh,
            // 2 kh + 1 (always lower-K + upper-K) and runs their epilogue
            f2_t own[2][8];
            {
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
                        own[mm][i] = kh ? f2_pack(other.x + mine.x, other.y + mine.y)
                                        : f2_pack(mine.x + other.x, mine.y + other.y);
                    }
            }
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
                float yhalf;
                {
                    const bool b4 = l8 & 4, b2 = l8 & 2, b1 = l8 & 1;
                    float y4[4];
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const float send = b4 ? yp[t] : yp[t + 4];
                        const float keep = b4 ? yp[t + 4] : yp[t];
                        y4[t] = keep + __shfl_xor_sync(kFull8, send, 4);
                    }
                    float y2[2];
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        const float send = b2 ? y4[t] : y4[t + 2];
                        const float keep = b2 ? y4[t + 2] : y4[t];
                        y2[t] = keep + __shfl_xor_sync(kFull8, send, 2);
                    }
                    const float send = b1 ? y2[0] : y2[1];
                    const float keep = b1 ? y2[1] : y2[0];
                    yhalf = keep + __shfl_xor_sync(kFull8, send, 1);
                }
                YX[kh * kBatchRows + rr_own] = yhalf;
                asm volatile("bar.sync %0, 64;" ::"r"(1 + wr) : "memory");
                const float yhat = YX[rr_own] + YX[kBatchRows + rr_own];
                const bool own_valid = rr_own < bsz;
                const float res = own_valid ? yhat - R0[rr_own] : 0.f;
                const float dy_own = (2.0f / (float)bsz) * res;
                if (!kh) lossacc = fmaf(res, res, lossacc);
                float dy[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) dy[i] = __shfl_sync(kFull8, dy_own, (lane & 24) | i);
                float2 gf[2], gb[2];
#pragma unroll
                for (int mm = 0; mm < 2; ++mm) {
                    const int jp = l8 + 8 * (2 * kh + mm);
                    const float2 fw = *reinterpret_cast<const float2 *>(F + 2 * jp);
                    gf[mm] = gb[mm] = make_float2(0.f, 0.f);
                    float *dzrow = DZ + jp * G::DS + 2 * (32 * wr + q);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const float2 a = f2_unpack(own[mm][i]);
                        const float2 z =
                            make_float2(a.x > 0.f ? dy[i] * fw.x : 0.f, a.y > 0.f ? dy[i] * fw.y : 0.f);
                        gf[mm].x = fmaf(a.x, dy[i], gf[mm].x);
                        gf[mm].y = fmaf(a.y, dy[i], gf[mm].y);
                        gb[mm].x += z.x;
                        gb[mm].y += z.y;
                        *reinterpret_cast<float2 *>(dzrow + 8 * i) = z;
                    }
                }
#pragma unroll
                for (int mm = 0; mm < 2; ++mm) {
                    gf[mm].x += __shfl_xor_sync(kFull8, gf[mm].x, 8);
                    gf[mm].y += __shfl_xor_sync(kFull8, gf[mm].y, 8);
                    gb[mm].x += __shfl_xor_sync(kFull8, gb[mm].x, 8);
                    gb[mm].y += __shfl_xor_sync(kFull8, gb[mm].y, 8);
                    gf[mm].x += __shfl_xor_sync(kFull8, gf[mm].x, 16);
                    gf[mm].y += __shfl_xor_sync(kFull8, gf[mm].y, 16);
                    gb[mm].x += __shfl_xor_sync(kFull8, gb[mm].x, 16);
                    gb[mm].y += __shfl_xor_sync(kFull8, gb[mm].y, 16);
                }
                if (q == 0) {
#pragma unroll
                    for (int mm = 0; mm < 2; ++mm) {
                        const int jp = l8 + 8 * (2 * kh + mm);
                        *reinterpret_cast<float2 *>(RED + wr * 128 + 2 * jp) = gf[mm];
                        *reinterpret_cast<float2 *>(RED + wr * 128 + 64 + 2 * jp) = gb[mm];
                    }
                }
            }
            __syncthreads();

            // ---- weight gradient gW = dZ^T X (hybrid_nn.cpp:109) --------------
            const int rh = q >> 1, jq = q & 1;
            f2_t ga[2][16];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int u = 0; u < 16; ++u) ga[i][u] = 0ull;
            {
                const float *zb = DZ + (4 * warp + jq) * G::DS + 2 * 64 * rh;
                const float *xb = X + 64 * rh * G::XS + 4 * l8;
#pragma unroll 1
                for (int r = 0; r < 64; r += 4) {
                    ulonglong2 z[2][2];
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        z[i][0] = *reinterpret_cast<const ulonglong2 *>(zb + 2 * i * G::DS + 2 * r);
                        z[i][1] = *reinterpret_cast<const ulonglong2 *>(zb + 2 * i * G::DS + 2 * r + 4);
                    }
#define NOMA_W8_GRAD(RR, ZP)                                                             \
    {                                                                                    \
        float4 xv[4];                                                                    \
        _Pragma("unroll") for (int gg = 0; gg < 4; ++gg)                                 \
            xv[gg] = *reinterpret_cast<const float4 *>(xb + (r + RR) * G::XS + 32 * gg); \
        _Pragma("unroll") for (int i = 0; i < 2; ++i)                                    \
            _Pragma("unroll") for (int gg = 0; gg < 4; ++gg) {                           \
            f2_fma(ga[i][4 * gg + 0], ZP, f2_bcast(xv[gg].x));                           \
            f2_fma(ga[i][4 * gg + 1], ZP, f2_bcast(xv[gg].y));                           \
            f2_fma(ga[i][4 * gg + 2], ZP, f2_bcast(xv[gg].z));                           \
            f2_fma(ga[i][4 * gg + 3], ZP, f2_bcast(xv[gg].w));                           \
        }                                                                                \
    }
                    NOMA_W8_GRAD(0, z[i][0].x)
                    NOMA_W8_GRAD(1, z[i][0].y)
                    NOMA_W8_GRAD(2, z[i][1].x)
                    NOMA_W8_GRAD(3, z[i][1].y)
#undef NOMA_W8_GRAD
                }
            }
            // the two row halves (lanes l and l ^ 16) add; each keeps 8 columns
            float2 gk[2][8];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const float2 send = f2_unpack(rh ? ga[i][u] : ga[i][u + 8]);
                    const float2 keep = f2_unpack(rh ? ga[i][u + 8] : ga[i][u]);
                    const float rx = __shfl_xor_sync(kFull8, send.x, 16);
                    const float ry = __shfl_xor_sync(kFull8, send.y, 16);
                    gk[i][u] = rh ? make_float2(rx + keep.x, ry + keep.y) : make_float2(keep.x + rx, keep.y + ry);
                }
            __syncthreads();  // X and DZ are dead

            // ---- next minibatch in flight while Adam runs ---------------------
            if (nb > 0) gather(nidx, nb);

            // ---- Adam (hybrid_nn.cpp:118-144), FP32 moments in registers -----
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int jp = 4 * warp + jq + 2 * i;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int uu = rh * 8 + u, c = 4 * l8 + 32 * (uu >> 2) + (uu & 3);
                    float2 *wp = reinterpret_cast<float2 *>(W2 + jp * G::WS + 2 * c);
                    float2 th = *wp;
                    const float2 gg = gk[i][u];
                    mw[i][u].x = p.b1 * mw[i][u].x + p.omb1 * gg.x;
                    mw[i][u].y = p.b1 * mw[i][u].y + p.omb1 * gg.y;
                    vw[i][u].x = p.b2 * vw[i][u].x + p.omb2 * (gg.x * gg.x);
                    vw[i][u].y = p.b2 * vw[i][u].y + p.omb2 * (gg.y * gg.y);
                    th.x -= adam_step(lrc * mw[i][u].x, vw[i][u].x * ic2, p.eps);
                    th.y -= adam_step(lrc * mw[i][u].y, vw[i][u].y * ic2, p.eps);
                    *wp = th;
                }
            }
            if (tid < 128) {  // biases (tid < 64) and final weights: fixed-order sum of the warps
                const int j = tid & 63, part = tid < 64 ? 64 : 0;
                const float gsum =
                    ((RED[part + j] + RED[128 + part + j]) + RED[256 + part + j]) + RED[384 + part + j];
                float *tp = tid < 64 ? B + j : F + j;
                mb = p.b1 * mb + p.omb1 * gsum;
                vb = p.b2 * vb + p.omb2 * (gsum * gsum);
                *tp -= adam_step(lrc * mb, vb * ic2, p.eps);
            }
            cp_wait_all();
            if (nb > 0) {
                w8_bar_wait(gbar, gphase);
                gphase ^= 1;
            }
            ++step;
            __syncthreads();
        }
        // ---- epoch loss (hybrid_nn.cpp:190-192): trace[e] = sum r^2 / n ------
        LS[tid] = lossacc;
        lossacc = 0.f;
        __syncthreads();
        if (tid == 0 && p.trace) {
            double s = 0.0;
            for (int i = 0; i < kW8Threads; ++i) s += LS[i];
            p.trace[(size_t)net * p.epochs + e] = s / (double)n;
        }
    }
    // ---- trained parameters out (FusedPlan layout) --------------------------
    float *po = p.plans + (size_t)net * g.plan_total;
    for (int i = tid; i < 64 * IN; i += kW8Threads) {
        const int j = i / IN, c = i % IN;
        po[g.plan_w[1] + j * g.plan_pad[0] + c] = W2[(j >> 1) * G::WS + 2 * c + (j & 1)];
    }
    if (tid < 64) {
        po[g.plan_b[1] + tid] = B[tid];
        po[g.plan_f + tid] = F[tid];
    }
}

// 1 hidden layer of 64, input 128, minibatch <= 128: the 8-warp kernel.
bool train_w8_fits(const TrainParams &p) {
    const NetGeom &g = p.g;
    if (std::getenv("NOMA_TRAIN_W8") && std::atoi(std::getenv("NOMA_TRAIN_W8")) == 0) return false;
    return g.nd == 2 && g.dims[1] == 64 && g.dims[0] == kW8In && p.batch >= 1 && p.batch <= kBatchRows &&
           p.rows <= 65535;
}

int train_w8_launch(TrainParams &p, cudaStream_t st) {
    const float *wide = p.design32;
    float *tmp = nullptr;
    if (p.layout == NOMA_LAYOUT_WIDEN_COMPLEX) {
        const size_t nrow_c = (size_t)(p.n_nets / p.K) * (p.rows / 2);
        if (cudaMallocAsync(&tmp, nrow_c * 2 * kW8In * sizeof(float), st) != cudaSuccess) return NOMA_ERR_CUDA;
        if (widen_rows_launch(p.design32, tmp, nrow_c, kW8In, st)) return NOMA_ERR_CUDA;
        wide = tmp;
    }
    cudaFuncSetAttribute(train_w8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)W8Geom::bytes);
    train_w8_kernel<<<p.n_nets, kW8Threads, W8Geom::bytes, st>>>(p, wide);
    const int rc = cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;
    if (tmp) cudaFreeAsync(tmp, st);
    p.mode = 4;
    return rc;
}

}  // namespace noma_dev
