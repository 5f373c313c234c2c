// Pilot-phase training, throughput mode, for one-hidden-layer nets of width 64
// (C1: dims [32,64]; C5: dims [64,64]): replaces hybrid_nn::train
// (hybrid_nn.cpp:158-195) with loss_and_grad (:84-114) and adam_step
// (:118-144) fused, one 4-warp CTA per user net, two or three nets per SM.
//
// Why a second throughput kernel (profiles/r02_*): the 16-warp kernel of
// k_train.cu runs one net per SM, so every non-GEMM phase of a step (gather,
// residual, final layer, Adam, barriers -- ~30 % of a C5 step) leaves the FMA
// pipe idle, and its 4x4 register tiles cost 0.75 shared-memory wavefronts
// per FFMA2 (smem-bound at 67 % of the FMA rate).  Here:
//   * a net needs 4 warps and ~88 KB (C5), so two nets share an SM and one
//     net's phases overlap the other's GEMMs;
//   * 8 x 8 FFMA2 register tiles (64 accumulators per thread): 0.375
//     wavefronts per FFMA2, both GEMMs (forward, weight gradient);
//   * Adam moments live in registers for the whole training: the thread that
//     finishes a weight-gradient element owns that parameter, so no gradient
//     buffer and no moment traffic;
//   * the minibatch is copied by one bulk copy per row (TMA engine, counted on
//     an mbarrier) from a pre-widened FP32 design
//     (rows 2t = [Re x_t; Im x_t], 2t+1 = [Im x_t; -Re x_t], iq_transform.cpp:
//     17-20) straight into a row-major tile while the previous step's Adam
//     runs -- no transposition, no registers;
//   * the forward keeps the activations in registers through the residual:
//     the final dot reduces over the warp (all 64 neurons of 32 rows), the
//     residual, dZ and the final-layer / bias gradients need no barrier.
//
// Layouts (floats, shared memory):
//   X   [128][IN+8]       minibatch rows, row-major (stride == 8 mod 32)
//   W2  [32][2*IN+4]      W2[jp][2c+e] = W[2jp+e][c]  (neuron pairs, FFMA2 lanes)
//   DZ  [32][2*128+8]     DZ[jp][2r+e] = dZ[2jp+e][r]
// Arithmetic is FP32 FMA (fma.rn.f32x2 = two IEEE FP32 FMAs); the frozen
// linear branch enters through r0 = y - X w0, precomputed in FP64 by the LLS
// kernel (as in k_train.cu).  Summation orders are fixed: bit-reproducible.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "kernels.cuh"
#include "tiles.cuh"

namespace noma_dev {

namespace {

constexpr int kW4Threads = 128;
constexpr unsigned kFull = 0xffffffffu;

template <int IN>
struct W4Geom {
    static constexpr int XS = IN + 8;                  // X row stride: == 8 mod 32, 4 rows = k x 128 B (TMA)
    static constexpr int WS = 2 * IN + 4;              // W2 row (neuron pair) stride
    static constexpr int DS = 2 * kBatchRows + 8;      // DZ row stride, == 8 mod 32
    static constexpr int off_x = 0;
    static constexpr int off_w = off_x + kBatchRows * XS;
    static constexpr int off_b = off_w + 32 * WS;
    static constexpr int off_f = off_b + 64;
    static constexpr int off_dz = off_f + 64;
    static constexpr int off_red = off_dz + 32 * DS;   // [warp][gf | gb][64]
    static constexpr int off_r0 = off_red + 4 * 2 * 64;
    static constexpr int off_loss = off_r0 + kBatchRows;
    static constexpr int off_gbar = off_loss + kBatchRows;  // 8-byte mbarrier (minibatch rows)
    static constexpr int off_end = off_gbar + 2;
    static constexpr size_t bytes = (size_t)off_end * sizeof(float);
};

__device__ __forceinline__ void cp4_zfill(float *dst, const float *src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(valid ? 4 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}
// minibatch rows by one bulk copy each (TMA engine) counted on an mbarrier:
// 128 copies per step instead of IN / 4 cp.async per thread
__device__ __forceinline__ uint32_t w4_s2u(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void w4_row_copy(float *dst, const float *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     w4_s2u(dst)),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
// four widened rows by one TMA gather (tile::gather4): box [XS floats x 1 row]
// per row over a [rows][IN] tensor map, so the XS - IN pad columns come back
// as out-of-bounds zeros and the tile keeps its padded row stride
__device__ __forceinline__ void w4_gather4(float *dst, const CUtensorMap *tm, int r0, int r1, int r2, int r3,
                                           uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(w4_s2u(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void w4_bar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W4_MBW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W4_MBW_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ float2 lo_hi(unsigned long long v) { return f2_unpack(v); }

}  // namespace

// Thread roles (q = lane >> 3, l8 = lane & 7):
//  forward   neuron pairs jp = l8 + 8m (m < 4), rows r_i = 32 warp + q + 4i (i < 8):
//            W reads 8-distinct per quarter, X reads quarter-uniform;
//  residual  lane l8 of a quarter owns row r_{l8} (exactly one thread per row);
//  gradient  neuron pairs jp = 8 warp + (q & 1) + 2i (i < 4), columns
//            c = 4 l8 + 32 g + t (g < IN/32, t < 4), rows of half q >> 1;
//            the two halves add through one lane-xor-16 exchange and each keeps
//            half of the columns: those parameters (and their Adam moments)
//            belong to the thread for the whole training.
template <int IN, bool G4>
__global__ void __launch_bounds__(kW4Threads, 2)
    train_w4_kernel(TrainParams p, const float *__restrict__ wide, const __grid_constant__ CUtensorMap tmap) {
    using G = W4Geom<IN>;
    constexpr int NG = IN / 32;  // 32-column groups per gradient thread
    constexpr int NU = 4 * NG;   // gradient columns per thread before the exchange
    constexpr int NK = NU / 2;   // columns kept after it
    extern __shared__ __align__(16) float sm[];
    const int net = blockIdx.x;
    if (p.status && p.status[net] != NOMA_OK) return;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, q = lane >> 3, l8 = lane & 7;
    const NetGeom &g = p.g;
    const int n = p.rows, d = net / p.K;
    float *X = sm + G::off_x;
    float *W2 = sm + G::off_w;
    float *B = sm + G::off_b;
    float *F = sm + G::off_f;
    float *DZ = sm + G::off_dz;
    float *RED = sm + G::off_red;
    float *R0 = sm + G::off_r0;
    float *LS = sm + G::off_loss;
    const bool clk_on = NOMA_PROBE_ON(p.clocks && blockIdx.x == 0 && threadIdx.x == 0);
    long long clk_acc[5] = {0, 0, 0, 0, 0}, clk_prev = clk_on ? clock64() : 0;
#define NOMA_W4_PHASE(I)                             \
    if (clk_on) {                                    \
        const long long now = clock64();             \
        clk_acc[I] += now - clk_prev;                \
        clk_prev = now;                              \
    }

    // ---- parameters in (FusedPlan layout, fused_inference.cpp:19-42) ------
    const float *pl = p.plans + (size_t)net * g.plan_total;
    for (int i = tid; i < 64 * IN; i += kW4Threads) {
        const int j = i / IN, c = i % IN;
        W2[(j >> 1) * G::WS + 2 * c + (j & 1)] = pl[g.plan_w[1] + j * g.plan_pad[0] + c];
    }
    if (tid < 64) {
        B[tid] = pl[g.plan_b[1] + tid];
        F[tid] = pl[g.plan_f + tid];
    }
    // Adam moments of the owned parameters (fresh state per train() call,
    // hybrid_nn.cpp:171)
    float2 mw[4][NK], vw[4][NK];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int u = 0; u < NK; ++u) mw[i][u] = vw[i][u] = make_float2(0.f, 0.f);
    float mb = 0.f, vb = 0.f;

    const uint16_t *permn = p.perm + (size_t)net * p.epochs * n;
    const float *wrow = wide + (size_t)d * n * IN;
    const float *r0n = p.r0 + (size_t)net * n;
    // minibatch copy (hybrid_nn.cpp:180-187): thread t copies widened row
    // perm[t] of the step (one bulk copy) and its r0 (cp.async, zero past the
    // batch end); rows past the batch end keep the previous, finite values --
    // their dZ is zero -- and start as zeros
    const uint32_t gbar = w4_s2u(sm + G::off_gbar);
    for (int i = tid; i < kBatchRows * G::XS; i += kW4Threads) X[i] = 0.0f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // before the bulk copies overwrite
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(gbar) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto gather = [&](int idx, int nrows) {  // every thread; nrows valid rows
        if constexpr (G4) {
            // groups of four rows; a short last group repeats its last valid
            // row (finite values with dZ = 0).  Lane 0 of each warp issues
            // its warp's groups.
            const int ng = (nrows + 3) >> 2;
            if (tid == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(gbar),
                             "r"((uint32_t)ng * 4 * G::XS * 4)
                             : "memory");
            const int grow = d * n + idx;
#pragma unroll
            for (int gq = 0; gq < 8; ++gq) {
                const int base = 32 * warp + 4 * gq;
                const int last = nrows - 1 - 32 * warp;
                const int r0 = __shfl_sync(kFull, grow, min(4 * gq, last));
                const int r1 = __shfl_sync(kFull, grow, min(4 * gq + 1, last));
                const int r2 = __shfl_sync(kFull, grow, min(4 * gq + 2, last));
                const int r3 = __shfl_sync(kFull, grow, min(4 * gq + 3, last));
                if (lane == 0 && base < nrows) w4_gather4(X + base * G::XS, &tmap, r0, r1, r2, r3, gbar);
            }
        } else {
            if (tid == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(gbar),
                             "r"((uint32_t)nrows * IN * 4)
                             : "memory");
            if (tid < nrows) w4_row_copy(X + tid * G::XS, wrow + (size_t)idx * IN, IN * 4, gbar);
        }
        cp4_zfill(R0 + tid, r0n + idx, tid < nrows);
    };
    uint32_t gphase = 0;
    {
        const int b0 = p.epochs > 0 ? min(p.batch, n) : 0;
        if (b0 > 0) {
            gather(tid < b0 ? permn[tid] : 0, b0);
            w4_bar_wait(gbar, gphase);
            gphase ^= 1;
        }
        cp_async_wait_all();
    }
    __syncthreads();

    float lossacc = 0.f;
    int step = 0;
    const int rr_own = 32 * warp + q + 4 * l8;  // residual row of this thread
    for (int e = 0; e < p.epochs; ++e) {
        for (int start = 0; start < n; start += p.batch) {
            const int bsz = min(p.batch, n - start);
            // next step's row index and this step's Adam constants, loaded early
            int ns = start + p.batch, ne = e;
            if (ns >= n) {
                ns = 0;
                ++ne;
            }
            const int nb = ne < p.epochs ? min(p.batch, n - ns) : 0;
            const int nidx = tid < nb ? permn[(size_t)ne * n + ns + tid] : 0;
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
            NOMA_W4_PHASE(0)

            // ---- forward: A = relu(W X + b) (hybrid_nn.cpp:60-67) ------------
            f2_t acc[4][8];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const f2_t bb = *reinterpret_cast<const f2_t *>(B + 2 * (l8 + 8 * m));
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[m][i] = bb;
            }
            {
                const float *wb = W2 + l8 * G::WS;
                const float *xb = X + (32 * warp + q) * G::XS;
#pragma unroll 1
                for (int k0 = 0; k0 < IN; k0 += 4) {
                    ulonglong2 w[4][2];
#pragma unroll
                    for (int m = 0; m < 4; ++m) {
                        w[m][0] = *reinterpret_cast<const ulonglong2 *>(wb + 8 * m * G::WS + 2 * k0);
                        w[m][1] = *reinterpret_cast<const ulonglong2 *>(wb + 8 * m * G::WS + 2 * k0 + 4);
                    }
                    float4 x[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) x[i] = *reinterpret_cast<const float4 *>(xb + 4 * i * G::XS + k0);
#define NOMA_W4_FWD(KK, WP)                                                    \
    _Pragma("unroll") for (int m = 0; m < 4; ++m)                              \
        _Pragma("unroll") for (int i = 0; i < 8; ++i)                          \
            f2_fma(acc[m][i], WP, f2_bcast(f4c<KK>(x[i])));
                    NOMA_W4_FWD(0, w[m][0].x)
                    NOMA_W4_FWD(1, w[m][0].y)
                    NOMA_W4_FWD(2, w[m][1].x)
                    NOMA_W4_FWD(3, w[m][1].y)
#undef NOMA_W4_FWD
                }
            }
            // ReLU; the final dot a . w_final (hybrid_nn.cpp:81) per row
            float yp[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) yp[i] = 0.f;
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const float2 fw = *reinterpret_cast<const float2 *>(F + 2 * (l8 + 8 * m));
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    float2 a = lo_hi(acc[m][i]);
                    a.x = fmaxf(a.x, 0.f);
                    a.y = fmaxf(a.y, 0.f);
                    acc[m][i] = f2_pack(a.x, a.y);
                    yp[i] = fmaf(fw.x, a.x, yp[i]);
                    yp[i] = fmaf(fw.y, a.y, yp[i]);
                }
            }
            NOMA_W4_PHASE(1)
            // reduce-scatter of the 8 row partials over the quarter's 8 lanes:
            // lane l8 ends with the full sum over all 64 neurons of row r_{l8}
            float yhat;
            {
                const bool b4 = l8 & 4, b2 = l8 & 2, b1 = l8 & 1;
                float y4[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const float send = b4 ? yp[t] : yp[t + 4];
                    const float keep = b4 ? yp[t + 4] : yp[t];
                    y4[t] = keep + __shfl_xor_sync(kFull, send, 4);
                }
                float y2[2];
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    const float send = b2 ? y4[t] : y4[t + 2];
                    const float keep = b2 ? y4[t + 2] : y4[t];
                    y2[t] = keep + __shfl_xor_sync(kFull, send, 2);
                }
                const float send = b1 ? y2[0] : y2[1];
                const float keep = b1 ? y2[1] : y2[0];
                yhat = keep + __shfl_xor_sync(kFull, send, 1);
            }
            // residual a.w_f - r0 = x w0 + a w_f - y (hybrid_nn.cpp:94), dy = 2r/B (:98)
            const bool own_valid = rr_own < bsz;
            const float res = own_valid ? yhat - R0[rr_own] : 0.f;
            const float dy_own = (2.0f / (float)bsz) * res;
            lossacc = fmaf(res, res, lossacc);
            float dy[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) dy[i] = __shfl_sync(kFull, dy_own, (lane & 24) | i);
            // dZ = (a > 0) ? dy w_f : 0 (:102, :107); g_final = a^T dy (:99);
            // g_b = colsum dZ (:110) -- partials over this thread's 8 rows
            float2 gf[4], gb[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const float2 fw = *reinterpret_cast<const float2 *>(F + 2 * (l8 + 8 * m));
                gf[m] = gb[m] = make_float2(0.f, 0.f);
                float *dzrow = DZ + (l8 + 8 * m) * G::DS + 2 * (32 * warp + q);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const float2 a = lo_hi(acc[m][i]);
                    const float2 z = make_float2(a.x > 0.f ? dy[i] * fw.x : 0.f, a.y > 0.f ? dy[i] * fw.y : 0.f);
                    gf[m].x = fmaf(a.x, dy[i], gf[m].x);
                    gf[m].y = fmaf(a.y, dy[i], gf[m].y);
                    gb[m].x += z.x;
                    gb[m].y += z.y;
                    *reinterpret_cast<float2 *>(dzrow + 8 * i) = z;
                }
            }
            // over the four quarters (rows), then one partial per warp
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                gf[m].x += __shfl_xor_sync(kFull, gf[m].x, 8);
                gf[m].y += __shfl_xor_sync(kFull, gf[m].y, 8);
                gb[m].x += __shfl_xor_sync(kFull, gb[m].x, 8);
                gb[m].y += __shfl_xor_sync(kFull, gb[m].y, 8);
                gf[m].x += __shfl_xor_sync(kFull, gf[m].x, 16);
                gf[m].y += __shfl_xor_sync(kFull, gf[m].y, 16);
                gb[m].x += __shfl_xor_sync(kFull, gb[m].x, 16);
                gb[m].y += __shfl_xor_sync(kFull, gb[m].y, 16);
            }
            if (q == 0) {
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    *reinterpret_cast<float2 *>(RED + warp * 128 + 2 * (l8 + 8 * m)) = gf[m];
                    *reinterpret_cast<float2 *>(RED + warp * 128 + 64 + 2 * (l8 + 8 * m)) = gb[m];
                }
            }
            __syncthreads();
            NOMA_W4_PHASE(2)

            // ---- weight gradient gW = dZ^T X (hybrid_nn.cpp:109) --------------
            const int rh = q >> 1, jq = q & 1;
            f2_t ga[4][NU];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int u = 0; u < NU; ++u) ga[i][u] = 0ull;
            {
                const float *zb = DZ + (8 * warp + jq) * G::DS + 2 * 64 * rh;
                const float *xb = X + 64 * rh * G::XS + 4 * l8;
#pragma unroll 1
                for (int r = 0; r < 64; r += 4) {
                    ulonglong2 z[4][2];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        z[i][0] = *reinterpret_cast<const ulonglong2 *>(zb + 2 * i * G::DS + 2 * r);
                        z[i][1] = *reinterpret_cast<const ulonglong2 *>(zb + 2 * i * G::DS + 2 * r + 4);
                    }
                    float4 xv[4][NG];
#pragma unroll
                    for (int rr = 0; rr < 4; ++rr)
#pragma unroll
                        for (int gg = 0; gg < NG; ++gg)
                            xv[rr][gg] = *reinterpret_cast<const float4 *>(xb + (r + rr) * G::XS + 32 * gg);
#define NOMA_W4_GRAD(RR, ZP)                                                               \
    _Pragma("unroll") for (int i = 0; i < 4; ++i)                                          \
        _Pragma("unroll") for (int gg = 0; gg < NG; ++gg) {                                \
        f2_fma(ga[i][4 * gg + 0], ZP, f2_bcast(xv[RR][gg].x));                             \
        f2_fma(ga[i][4 * gg + 1], ZP, f2_bcast(xv[RR][gg].y));                             \
        f2_fma(ga[i][4 * gg + 2], ZP, f2_bcast(xv[RR][gg].z));                             \
        f2_fma(ga[i][4 * gg + 3], ZP, f2_bcast(xv[RR][gg].w));                             \
    }
                    NOMA_W4_GRAD(0, z[i][0].x)
                    NOMA_W4_GRAD(1, z[i][0].y)
                    NOMA_W4_GRAD(2, z[i][1].x)
                    NOMA_W4_GRAD(3, z[i][1].y)
#undef NOMA_W4_GRAD
                }
            }
            // the two row halves (lanes l and l ^ 16) add; each keeps NK columns
            float2 gk[4][NK];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int u = 0; u < NK; ++u) {
                    const float2 send = lo_hi(rh ? ga[i][u] : ga[i][u + NK]);
                    const float2 keep = lo_hi(rh ? ga[i][u + NK] : ga[i][u]);
                    const float rx = __shfl_xor_sync(kFull, send.x, 16);
                    const float ry = __shfl_xor_sync(kFull, send.y, 16);
                    // fixed order: row half 0 + row half 1
                    gk[i][u] = rh ? make_float2(rx + keep.x, ry + keep.y) : make_float2(keep.x + rx, keep.y + ry);
                }
            __syncthreads();  // X and DZ are dead
            NOMA_W4_PHASE(3)

            // ---- next minibatch in flight while Adam runs ---------------------
            if (nb > 0) gather(nidx, nb);

            // ---- Adam (hybrid_nn.cpp:118-144), FP32 moments in registers -----
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int jp = 8 * warp + jq + 2 * i;
#pragma unroll
                for (int u = 0; u < NK; ++u) {
                    const int uu = rh * NK + u, c = 4 * l8 + 32 * (uu >> 2) + (uu & 3);
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
            {  // biases (tid < 64) and final weights: fixed-order sum of the warps
                const int j = tid & 63, part = tid < 64 ? 64 : 0;
                const float gsum = ((RED[part + j] + RED[128 + part + j]) + RED[256 + part + j]) + RED[384 + part + j];
                float *tp = tid < 64 ? B + j : F + j;
                mb = p.b1 * mb + p.omb1 * gsum;
                vb = p.b2 * vb + p.omb2 * (gsum * gsum);
                *tp -= adam_step(lrc * mb, vb * ic2, p.eps);
            }
            cp_async_wait_all();
            if (nb > 0) {
                w4_bar_wait(gbar, gphase);
                gphase ^= 1;
            }
            ++step;
            __syncthreads();
            NOMA_W4_PHASE(4)
        }
        // ---- epoch loss (hybrid_nn.cpp:190-192): trace[e] = sum r^2 / n ------
        LS[tid] = lossacc;
        lossacc = 0.f;
        __syncthreads();
        if (tid == 0 && p.trace) {
            double s = 0.0;
            for (int i = 0; i < kW4Threads; ++i) s += LS[i];
            p.trace[(size_t)net * p.epochs + e] = s / (double)n;
        }
    }
    if (clk_on)
        for (int i = 0; i < 5; ++i) p.clocks[i] = clk_acc[i];
#undef NOMA_W4_PHASE
    // ---- trained parameters out (FusedPlan layout) --------------------------
    float *po = p.plans + (size_t)net * g.plan_total;
    for (int i = tid; i < 64 * IN; i += kW4Threads) {
        const int j = i / IN, c = i % IN;
        po[g.plan_w[1] + j * g.plan_pad[0] + c] = W2[(j >> 1) * G::WS + 2 * c + (j & 1)];
    }
    if (tid < 64) {
        po[g.plan_b[1] + tid] = B[tid];
        po[g.plan_f + tid] = F[tid];
    }
}

// Widened FP32 design rows for the minibatch gather: row 2t = [Re x_t | Im x_t]
// (the LLS kernel's FP32 copy), row 2t+1 = [Im x_t | -Re x_t].
__global__ void widen_rows_kernel(const float *__restrict__ d32, float *__restrict__ wide, size_t nrow_c,
                                  int width) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nrow_c * width) return;
    const size_t t = i / width;
    const int c = (int)(i % width), M = width / 2;
    const float *row = d32 + t * width;
    wide[2 * t * width + c] = row[c];
    wide[(2 * t + 1) * width + c] = c < M ? row[M + c] : -row[c - M];
}

int widen_rows_launch(const float *d32, float *wide, size_t nrow_c, int width, cudaStream_t st) {
    const size_t tot = nrow_c * width;
    if (tot == 0) return NOMA_OK;
    widen_rows_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(d32, wide, nrow_c, width);
    return cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;
}

bool tensor_map_encode_tiled(CUtensorMap *tm, CUtensorMapDataType dt, int rank, void *base, const cuuint64_t *gdim,
                             const cuuint64_t *gstride, const cuuint32_t *box, const cuuint32_t *estride) {
    using Fn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                            const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                            CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Fn fn = [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<Fn>(f);
    }();
    if (!fn) return false;
    return fn(tm, dt, (cuuint32_t)rank, base, gdim, gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 1 hidden layer of 64, input 32 or 64, minibatch <= 128: the 4-warp kernel.
bool train_w4_fits(const TrainParams &p) {
    const NetGeom &g = p.g;
    if (std::getenv("NOMA_TRAIN_W4") && std::atoi(std::getenv("NOMA_TRAIN_W4")) == 0) return false;
    return g.nd == 2 && g.dims[1] == 64 && (g.dims[0] == 32 || g.dims[0] == 64) && p.batch >= 1 &&
           p.batch <= kBatchRows && p.rows <= 65535;
}

int train_w4_launch(TrainParams &p, cudaStream_t st) {
    const int IN = p.g.dims[0];
    const float *wide = p.design32;
    float *tmp = nullptr;
    if (p.layout == NOMA_LAYOUT_WIDEN_COMPLEX) {
        const size_t nrow_c = (size_t)(p.n_nets / p.K) * (p.rows / 2);
        if (cudaMallocAsync(&tmp, nrow_c * 2 * IN * sizeof(float), st) != cudaSuccess) return NOMA_ERR_CUDA;
        const size_t tot = nrow_c * IN;
        widen_rows_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(p.design32, tmp, nrow_c, IN);
        wide = tmp;
    }
    int rc = NOMA_OK;
    // tensor map over the widened rows [designs * rows][IN] for the gather4
    // path (NOMA_W4_GATHER4=0: one bulk copy per row)
    CUtensorMap tmap;
    std::memset(&tmap, 0, sizeof(tmap));
    const char *ge = std::getenv("NOMA_W4_GATHER4");
    bool g4 = !(ge && std::atoi(ge) == 0);
    const size_t total_rows = (size_t)((p.n_nets + p.K - 1) / p.K) * p.rows;
    if (g4 && total_rows > 0x7fffffffu) g4 = false;
    if (g4) {
        const int XS = IN == 32 ? W4Geom<32>::XS : W4Geom<64>::XS;
        const cuuint64_t gdim[2] = {(cuuint64_t)IN, (cuuint64_t)total_rows};
        const cuuint64_t gstride[1] = {(cuuint64_t)IN * sizeof(float)};
        const cuuint32_t box[2] = {(cuuint32_t)XS, 1};
        const cuuint32_t estr[2] = {1, 1};
        g4 = tensor_map_encode_tiled(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(wide), gdim,
                                     gstride, box, estr);
    }
    auto go = [&](auto kern, size_t smem) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<p.n_nets, kW4Threads, smem, st>>>(p, wide, tmap);
        rc = cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;
    };
    if (IN == 32)
        g4 ? go(train_w4_kernel<32, true>, W4Geom<32>::bytes) : go(train_w4_kernel<32, false>, W4Geom<32>::bytes);
    else
        g4 ? go(train_w4_kernel<64, true>, W4Geom<64>::bytes) : go(train_w4_kernel<64, false>, W4Geom<64>::bytes);
    if (tmp) cudaFreeAsync(tmp, st);
    p.mode = 3;
    return rc;
}

}  // namespace noma_dev
