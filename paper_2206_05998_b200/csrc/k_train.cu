// Pilot-phase training on sm_100a: replaces hybrid_nn::train
// (hybrid_nn.cpp:158-195) together with loss_and_grad (:84-114) and
// adam_step (:118-144) -- one fused kernel, one CTA (8 warps) per user
// network, for all epochs x minibatches.
//
// On-chip state for the whole training (never leaves the SM):
//   * weights, biases, final layer      -- shared memory (FP32)
//   * gradients (1-2 split partials)    -- shared memory (FP32)
//   * Adam first/second moments         -- shared memory (registers if short)
//   * minibatch input and activations   -- shared memory, feature-major
// Per minibatch: gather the shuffled rows straight from the (L2-resident)
// design -- the IQ-symmetry widening (iq_transform.cpp:17-20) is applied at
// load: odd widened rows are [Im; -Re] of the stored complex row -- then
// forward (final-layer dot fused into the last hidden layer's epilogue),
// residual, backward and the Adam update, separated by CTA barriers.  The
// dense contractions use the 8x4 FFMA register tiles of tiles.cuh.
//
// Frozen linear branch: w0 never changes during training (hybrid_nn.cpp:
// 129-144 never touches it), so the LLS kernel precomputes r0 = y - X w0 in
// FP64 once per row and the network trains its ReLU branch on a_N w - r0.
// This is the reference loss exactly (residual = x w0 + a_N w - y,
// hybrid_nn.cpp:94) without the FP32 cancellation of x w0 - y.
#include <math.h>
#include <cstdlib>

#include "kernels.cuh"
#include "tiles.cuh"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace noma_dev {

constexpr int kMaxSplit = 2;  // weight-gradient split-K partials

__device__ __forceinline__ void cp_async16_g2s(float *dst, const float *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async4_g2s(float *dst, const float *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all_g2s() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// Two CTA shapes: 16 warps with 4x4 FFMA2 tiles (one net per SM: large nets)
// and 8 warps with 8x4 FFMA2 tiles (two nets per SM when they fit: small
// nets); the tile width picks the final-layer partial block (16 / 32 j).
template <int NT>
__host__ __device__ constexpr int yp_block() { return NT == 512 ? 16 : 32; }

template <int NT>
__host__ __device__ inline int grad_splits(int J, int C, int max_split) {
    const int tiles = NT == 512 ? (J >> 5) * (C >> 4) : (J >> 5) * (C >> 5);
    return tiles < NT / 32 ? max_split : 1;
}

// CS > 1: latency mode -- a thread-block cluster of CS CTAs trains one net.
// CTA `rank` owns minibatch rows [rank*RB, (rank+1)*RB), RB = 128/CS; each
// step the CTAs' weight-gradient partials are reduce-scattered through
// distributed shared memory (fixed summation order: deterministic), every CTA
// runs Adam on its 1/CS parameter slice and pushes the updated slice into all
// CTAs' weight copies, bracketed by two cluster barriers.
template <int NT, int NSLOT, int MINB, int CS>
__global__ void __launch_bounds__(NT, MINB) train_kernel(TrainParams p) {
    constexpr int kTrainThreads = NT;
    constexpr int kTrainWarps = NT / 32;
    constexpr int RB = kBatchRows / CS;  // minibatch rows per CTA
    extern __shared__ __align__(16) float sm[];
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = CS > 1 ? (int)cluster.block_rank() : 0;
    const int net = blockIdx.x / CS;
    if (p.status && p.status[net] != NOMA_OK) return;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const NetGeom &g = p.g;
    const int N = g.nd - 1;  // hidden layers
    const int n = p.rows, d = net / p.K;
    const int gstride = p.gs_stride;  // floats between gradient split partials
    float *XT = sm + p.off_x;
    float *PS = sm + p.off_ps;
    float *GS = sm + p.off_gs;
    float *r0b = sm + p.off_r0b;
    float *dy = sm + p.off_dy;
    float *red = sm + p.off_red;    // 128 floats: epoch loss reduction
    float *misc = sm + p.off_misc;  // [0] lr/corr1, [1] 1/corr2
    float *yp = sm + p.off_yp;      // [fp_N/32][128] final-layer partials
    // optional phase-cycle instrumentation (block 0, thread 0; NOMA_PHASE_CLOCKS)
    const bool clk_on = NOMA_PROBE_ON(p.clocks && blockIdx.x == 0 && threadIdx.x == 0);
    long long clk_acc[6] = {0, 0, 0, 0, 0, 0}, clk_prev = clk_on ? clock64() : 0;
#define NOMA_PHASE(I)                                \
    if (clk_on) {                                    \
        const long long now = clock64();             \
        clk_acc[I] += now - clk_prev;                \
        clk_prev = now;                              \
    }

    for (int i = tid; i < p.off_end; i += kTrainThreads) sm[i] = 0.0f;
    __syncthreads();
    const float *pl = p.plans + (size_t)net * g.plan_total;
    for (int l = 1; l <= N; ++l) {
        const int rowsl = g.dims[l], cols = g.dims[l - 1];
        for (int i = tid; i < rowsl * cols; i += kTrainThreads) {
            const int j = i / cols, c = i % cols;
            PS[g.pw[l] + j * g.sw[l] + c] = pl[g.plan_w[l] + j * g.plan_pad[l - 1] + c];
        }
        for (int j = tid; j < rowsl; j += kTrainThreads) PS[g.pb[l] + j] = pl[g.plan_b[l] + j];
    }
    for (int j = tid; j < g.dims[N]; j += kTrainThreads) PS[g.pf + j] = pl[g.plan_f + j];

    float mom1[NSLOT > 0 ? NSLOT : 1], mom2[NSLOT > 0 ? NSLOT : 1];
#pragma unroll
    for (int s = 0; s < NSLOT; ++s) mom1[s] = mom2[s] = 0.0f;
    __syncthreads();

    const int width = p.width, M = width / 2;
    const bool vec4 = (width & 3) == 0 && (M & 3) == 0;
    const int fpN = g.fp[N];
    const int njb = fpN / yp_block<NT>();  // final-layer partial blocks
    float *AN = N ? sm + p.off_a[N] : XT;
    float loss_acc = 0.0f;     // per-row-thread partial of the epoch loss
    long step = 0;
    // next-minibatch staging (two layers, 32-wide input, >= 8 warps idle in the
    // first layer's weight gradient -- the C2 shape): those warps cp.async the
    // next step's raw design rows and r0 into a_2, which is dead from then
    // until the next forward; the gather then only widens shared memory
    const bool stage_next = NT == 512 && CS == 1 && N >= 2 && width == 32 && vec4 &&
                            (g.fp[1] >> 5) * (g.fp[0] >> 4) * grad_splits<NT>(g.fp[1], g.fp[0], p.gsplit) <=
                                kTrainWarps - 8 &&
                            g.fp[2] * kSR >= kBatchRows * (32 + 2);
    float *stg = N >= 2 ? sm + p.off_a[2] : nullptr;  // [128][32] rows, then r0[128], idx[128]
    const bool stage_warp = warp >= kTrainWarps - 8;
    for (int e = 0; e < p.epochs; ++e) {
        const uint16_t *perm = p.perm + ((size_t)net * p.epochs + e) * n;
        for (int start = 0; start < n; start += p.batch) {
            const int bsz = min(p.batch, n - start);
            NOMA_PHASE(5)
            if (stage_next && step > 0) {  // rows staged in a_2 during the previous step
                const int r = tid & (kBatchRows - 1), h = tid >> 7;  // 4 threads per row
                const float *row = stg + r * 32;
                const int idx = reinterpret_cast<const int *>(stg + kBatchRows * 33)[r];
                const bool odd = p.layout == NOMA_LAYOUT_WIDEN_COMPLEX && idx >= 0 && (idx & 1);
                if (h == 0) r0b[r] = stg[kBatchRows * 32 + r];
#pragma unroll
                for (int c = h * 4; c < 32; c += 16) {
                    float4 v;
                    if (idx < 0) v = make_float4(0.f, 0.f, 0.f, 0.f);
                    else if (!odd) v = *reinterpret_cast<const float4 *>(row + c);
                    else if (c < M) v = *reinterpret_cast<const float4 *>(row + M + c);
                    else {
                        const float4 t = *reinterpret_cast<const float4 *>(row + c - M);
                        v = make_float4(-t.x, -t.y, -t.z, -t.w);
                    }
                    XT[c * kSR + r] = v.x;
                    XT[(c + 1) * kSR + r] = v.y;
                    XT[(c + 2) * kSR + r] = v.z;
                    XT[(c + 3) * kSR + r] = v.w;
                }
                if (tid == kTrainThreads - 1) {
                    if (p.atab) {
                        misc[0] = p.atab[2 * step];
                        misc[1] = p.atab[2 * step + 1];
                    } else {
                        const double c1 = 1.0 - pow(p.b1d, (double)(step + 1));
                        const double c2 = 1.0 - pow(p.b2d, (double)(step + 1));
                        misc[0] = (float)(p.lr_d / c1);
                        misc[1] = (float)(1.0 / c2);
                    }
                }
            } else
            // ---- gather (IQ widening at load): NT/128 threads per batch row -
            {
                constexpr int TPR = NT / kBatchRows;
                const int r = tid & (kBatchRows - 1), h = tid >> 7;
                const int rg = rank * RB + r;  // row of the minibatch (CS > 1: r < RB local)
                if (r < RB && rg < bsz) {
                    const int idx = perm[start + rg];
                    if (h == 0) r0b[r] = p.r0[(size_t)net * n + idx];
                    const bool wid = p.layout == NOMA_LAYOUT_WIDEN_COMPLEX;
                    const float *src = wid ? p.design32 + ((size_t)d * (n >> 1) + (idx >> 1)) * width
                                           : p.design32 + ((size_t)d * n + idx) * width;
                    const bool odd = wid && (idx & 1);
                    if (vec4) {
                        for (int c = h * 4; c < width; c += 4 * TPR) {
                            float4 v;
                            if (!odd) {
                                v = *reinterpret_cast<const float4 *>(src + c);
                            } else if (c < M) {
                                v = *reinterpret_cast<const float4 *>(src + M + c);
                            } else {
                                const float4 t = *reinterpret_cast<const float4 *>(src + c - M);
                                v = make_float4(-t.x, -t.y, -t.z, -t.w);
                            }
                            XT[c * kSR + r] = v.x;
                            XT[(c + 1) * kSR + r] = v.y;
                            XT[(c + 2) * kSR + r] = v.z;
                            XT[(c + 3) * kSR + r] = v.w;
                        }
                    } else {
                        for (int c = h; c < width; c += TPR)
                            XT[c * kSR + r] = !odd ? src[c] : (c < M ? src[M + c] : -src[c - M]);
                    }
                } else {
                    if (h == 0) r0b[r] = 0.0f;
                    for (int c = h; c < width; c += TPR) XT[c * kSR + r] = 0.0f;
                }
                if (tid == kTrainThreads - 1) {  // Adam constants for this step
                    if (p.atab) {  // precomputed (adam_table_kernel)
                        misc[0] = p.atab[2 * step];
                        misc[1] = p.atab[2 * step + 1];
                    } else {       // FP64 pow, hybrid_nn.cpp:133-135
                        const double c1 = 1.0 - pow(p.b1d, (double)(step + 1));
                        const double c2 = 1.0 - pow(p.b2d, (double)(step + 1));
                        misc[0] = (float)(p.lr_d / c1);
                        misc[1] = (float)(1.0 / c2);
                    }
                }
            }
            __syncthreads();
            NOMA_PHASE(0)
            // ---- forward (hybrid_nn.cpp:60-72); last layer also forms yp -----
            for (int l = 1; l <= N; ++l) {
                const float *ain = l == 1 ? XT : sm + p.off_a[l - 1];
                const float *wfp = l == N ? PS + g.pf : nullptr;
                float *ypp = l == N ? yp : nullptr;
                if constexpr (NT == 512)
                    tile_forward44<kTrainWarps>(PS + g.pw[l], g.sw[l], PS + g.pb[l], ain,
                                                sm + p.off_a[l], g.fp[l], g.fp[l - 1], warp, lane,
                                                wfp, ypp, RB);
                else
                    tile_forward<kTrainWarps>(PS + g.pw[l], g.sw[l], PS + g.pb[l], ain,
                                              sm + p.off_a[l], g.fp[l], g.fp[l - 1], warp, lane,
                                              wfp, ypp);
                __syncthreads();
            }
            NOMA_PHASE(1)
            // ---- residual a_N w - r0, dy = 2 r / B (hybrid_nn.cpp:94-98) ------
            if (tid < kBatchRows) {
                float yhat = 0.0f;
                if (N) {
                    for (int b = 0; b < njb; ++b) yhat += yp[b * kBatchRows + tid];
                } else {
                    const float *wf = PS + g.pf;
                    for (int j = 0; j < fpN; ++j) yhat = fmaf(XT[j * kSR + tid], wf[j], yhat);
                }
                const float res = (tid < RB && rank * RB + tid < bsz) ? yhat - r0b[tid] : 0.0f;
                dy[tid] = (2.0f / (float)bsz) * res;
                loss_acc = fmaf(res, res, loss_acc);
            }
            __syncthreads();
            NOMA_PHASE(2)
            // ---- final layer gradient and dZ_N (hybrid_nn.cpp:99-107) --------
            {
                // item (j, part): neuron j, rows 4 part + 32 c + e (c, e < 4) as
                // four float4 chunks -- a quarter-warp reads 128 contiguous
                // bytes (conflict-free), the 16 values stay in registers for
                // both the gradient sum and dZ_N
                const float *wf = PS + g.pf;
                for (int it = tid; it < fpN * 8; it += kTrainThreads) {  // fpN*8 % 256 == 0
                    const int j = it >> 3, part = it & 7;
                    float4 *row = reinterpret_cast<float4 *>(AN + j * kSR + 4 * part);
                    const float4 *dyp = reinterpret_cast<const float4 *>(dy + 4 * part);
                    float4 a[4], y[4];
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        a[c] = row[8 * c];
                        y[c] = dyp[8 * c];
                    }
                    float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        s4[0] = fmaf(a[c].x, y[c].x, s4[0]);
                        s4[1] = fmaf(a[c].y, y[c].y, s4[1]);
                        s4[2] = fmaf(a[c].z, y[c].z, s4[2]);
                        s4[3] = fmaf(a[c].w, y[c].w, s4[3]);
                    }
                    float s = (s4[0] + s4[1]) + (s4[2] + s4[3]);
                    s += __shfl_xor_sync(0xffffffffu, s, 1);
                    s += __shfl_xor_sync(0xffffffffu, s, 2);
                    s += __shfl_xor_sync(0xffffffffu, s, 4);
                    if (part == 0) GS[g.pf + j] = s;
                    if (N) {
                        // dZ_N, and its row sum = the top layer's bias gradient
                        // (:110; the top layer's weight-gradient tiles skip it,
                        // which evens their per-warp work)
                        const float wj = wf[j];
                        float b4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const float4 z = make_float4(a[c].x > 0.0f ? y[c].x * wj : 0.0f, a[c].y > 0.0f ? y[c].y * wj : 0.0f,
                                                         a[c].z > 0.0f ? y[c].z * wj : 0.0f, a[c].w > 0.0f ? y[c].w * wj : 0.0f);
                            row[8 * c] = z;
                            b4[0] += z.x;
                            b4[1] += z.y;
                            b4[2] += z.z;
                            b4[3] += z.w;
                        }
                        float b = (b4[0] + b4[1]) + (b4[2] + b4[3]);
                        b += __shfl_xor_sync(0xffffffffu, b, 1);
                        b += __shfl_xor_sync(0xffffffffu, b, 2);
                        b += __shfl_xor_sync(0xffffffffu, b, 4);
                        if (part == 0) {
                            GS[g.pb[N] + j] = b;
                            if (p.gsplit > 1) GS[gstride + g.pb[N] + j] = 0.0f;
                        }
                    }
                }
            }
            __syncthreads();
            NOMA_PHASE(3)
            // ---- backward (hybrid_nn.cpp:105-112) ----------------------------
            for (int l = N; l >= 1; --l) {
                const float *ain = l == 1 ? XT : sm + p.off_a[l - 1];
                const int splits = grad_splits<NT>(g.fp[l], g.fp[l - 1], p.gsplit);
                if constexpr (NT == 512) {
                    // fewer tasks than warps (C2's first layer: 8 for 16): the idle
                    // warps sum the bias gradient (row sums of dZ_l, :110), so the
                    // tile tasks carry no bias work and finish together
                    const int ntask = (g.fp[l] >> 5) * (g.fp[l - 1] >> 4) * splits;
                    const bool idle_bias = l != N && ntask < kTrainWarps;
                    tile_weight_grad44<kTrainWarps>(sm + p.off_a[l], ain, GS + g.pw[l], g.sw[l],
                                                    GS + g.pb[l], g.fp[l], g.fp[l - 1], splits,
                                                    gstride, warp, lane, RB, l != N && !idle_bias);
                    if (stage_next && l == 1 && stage_warp) {  // the next minibatch's rows -> a_2
                        int ns = start + p.batch, ne = e;
                        if (ns >= n) {
                            ns = 0;
                            ++ne;
                        }
                        const int pt = tid - (kTrainWarps - 8) * 32;
                        const int r = pt & (kBatchRows - 1), hh = pt >> 7;  // half a row per thread
                        const int nb = ne < p.epochs ? min(p.batch, n - ns) : 0;
                        int *sidx = reinterpret_cast<int *>(stg + kBatchRows * 33);
                        if (r < nb) {
                            const int idx = p.perm[((size_t)net * p.epochs + ne) * n + ns + r];
                            const bool wid = p.layout == NOMA_LAYOUT_WIDEN_COMPLEX;
                            const float *src = wid ? p.design32 + ((size_t)d * (n >> 1) + (idx >> 1)) * width
                                                   : p.design32 + ((size_t)d * n + idx) * width;
#pragma unroll
                            for (int q = 0; q < 4; ++q) cp_async16_g2s(stg + r * 32 + 16 * hh + 4 * q, src + 16 * hh + 4 * q);
                            if (hh == 0) {
                                cp_async4_g2s(stg + kBatchRows * 32 + r, p.r0 + (size_t)net * n + idx);
                                sidx[r] = idx;
                            }
                        } else if (hh == 0) {
                            stg[kBatchRows * 32 + r] = 0.0f;
                            sidx[r] = -1;
                        }
                    }
                    if (idle_bias && warp >= ntask) {
                        const int nth = (kTrainWarps - ntask) * 32, t0 = tid - ntask * 32;
                        const float *dzl = sm + p.off_a[l];
                        for (int j = t0; j < g.fp[l]; j += nth) {
                            float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
                            for (int r = 0; r < RB; r += 4) {
                                const float4 z = *reinterpret_cast<const float4 *>(dzl + j * kSR + r);
                                s4.x += z.x;
                                s4.y += z.y;
                                s4.z += z.z;
                                s4.w += z.w;
                            }
                            GS[g.pb[l] + j] = (s4.x + s4.y) + (s4.z + s4.w);
                            if (p.gsplit > 1) GS[gstride + g.pb[l] + j] = 0.0f;
                        }
                    }
                } else
                    tile_weight_grad<kTrainWarps>(sm + p.off_a[l], ain, GS + g.pw[l], g.sw[l],
                                                  GS + g.pb[l], g.fp[l], g.fp[l - 1], splits,
                                                  gstride, warp, lane, l != N);
                __syncthreads();
                if (l > 1) {
                    if constexpr (NT == 512)
                        tile_backward_data44<kTrainWarps>(PS + g.pw[l], g.sw[l], sm + p.off_a[l],
                                                          sm + p.off_a[l - 1], g.fp[l - 1],
                                                          g.fp[l], warp, lane, RB);
                    else
                        tile_backward_data<kTrainWarps>(PS + g.pw[l], g.sw[l], sm + p.off_a[l],
                                                        sm + p.off_a[l - 1], g.fp[l - 1], g.fp[l],
                                                        warp, lane);
                    __syncthreads();
                }
            }
            NOMA_PHASE(4)
            // ---- Adam (hybrid_nn.cpp:118-144): FP32 moments, registers or smem
            {
                const float lrc = misc[0], ic2 = misc[1];
                if constexpr (CS > 1) {
                    // reduce-scatter the CS gradient partials over DSMEM, Adam on
                    // this CTA's slice, push the slice into every CTA's weights
                    cluster.sync();
                    float *M1 = sm + p.off_mom, *M2 = M1 + gstride;
                    const int slice = pad_to((g.ptotal + CS - 1) / CS, 4);
                    const int lo = rank * slice, hi = min(g.ptotal, lo + slice);
                    const float *gsr[CS];
                    float *psr[CS];
#pragma unroll
                    for (int q = 0; q < CS; ++q) {
                        gsr[q] = cluster.map_shared_rank(GS, q);
                        psr[q] = cluster.map_shared_rank(PS, q);
                    }
                    for (int i = lo + tid; i < hi; i += kTrainThreads) {
                        float gi = 0.0f;
#pragma unroll
                        for (int q = 0; q < CS; ++q) {
                            gi += gsr[q][i];
                            if (p.gsplit > 1) gi += gsr[q][gstride + i];
                        }
                        const float m1 = p.b1 * M1[i] + p.omb1 * gi;
                        const float m2 = p.b2 * M2[i] + p.omb2 * (gi * gi);
                        M1[i] = m1;
                        M2[i] = m2;
                        const float th = PS[i] - adam_step(lrc * m1, m2 * ic2, p.eps);
#pragma unroll
                        for (int q = 0; q < CS; ++q) psr[q][i] = th;
                    }
                    cluster.sync();
                } else if constexpr (NSLOT > 0) {
#pragma unroll
                    for (int s = 0; s < NSLOT; ++s) {
                        const int i = tid + s * kTrainThreads;
                        if (i < g.ptotal) {
                            // fixed-order sum of the split-K partials
                            const float gi = p.gsplit > 1 ? GS[i] + GS[gstride + i] : GS[i];
                            mom1[s] = p.b1 * mom1[s] + p.omb1 * gi;
                            mom2[s] = p.b2 * mom2[s] + p.omb2 * (gi * gi);
                            PS[i] -= adam_step(lrc * mom1[s], mom2[s] * ic2, p.eps);
                        }
                    }
                } else {
                    // moments interleaved (m1, m2) per parameter; two parameters
                    // per iteration: float2 gradients / parameters, float4
                    // moments (the regions are 16-byte aligned, padded to 4)
                    float *M12 = sm + p.off_mom;
                    const int npair = g.ptotal >> 1;
                    for (int t = tid; t < npair; t += kTrainThreads) {
                        float2 gi = *reinterpret_cast<const float2 *>(GS + 2 * t);
                        if (p.gsplit > 1) {
                            const float2 g2 = *reinterpret_cast<const float2 *>(GS + gstride + 2 * t);
                            gi.x += g2.x;
                            gi.y += g2.y;
                        }
                        float4 m = *reinterpret_cast<const float4 *>(M12 + 4 * t);
                        m.x = p.b1 * m.x + p.omb1 * gi.x;
                        m.y = p.b2 * m.y + p.omb2 * (gi.x * gi.x);
                        m.z = p.b1 * m.z + p.omb1 * gi.y;
                        m.w = p.b2 * m.w + p.omb2 * (gi.y * gi.y);
                        *reinterpret_cast<float4 *>(M12 + 4 * t) = m;
                        float2 th = *reinterpret_cast<const float2 *>(PS + 2 * t);
                        th.x -= adam_step(lrc * m.x, m.y * ic2, p.eps);
                        th.y -= adam_step(lrc * m.z, m.w * ic2, p.eps);
                        *reinterpret_cast<float2 *>(PS + 2 * t) = th;
                    }
                    if ((g.ptotal & 1) && tid == 0) {  // odd count: the last parameter
                        const int i = g.ptotal - 1;
                        const float gi = p.gsplit > 1 ? GS[i] + GS[gstride + i] : GS[i];
                        const float m1 = p.b1 * M12[2 * i] + p.omb1 * gi;
                        const float m2 = p.b2 * M12[2 * i + 1] + p.omb2 * (gi * gi);
                        M12[2 * i] = m1;
                        M12[2 * i + 1] = m2;
                        PS[i] -= adam_step(lrc * m1, m2 * ic2, p.eps);
                    }
                }
            }
            if (stage_next && stage_warp) cp_async_wait_all_g2s();  // staged rows land before the barrier
            ++step;
            __syncthreads();
        }
        // ---- epoch loss (hybrid_nn.cpp:190-192): trace[e] = sum r^2 / n ------
        if (tid < kBatchRows) red[tid] = loss_acc;
        loss_acc = 0.0f;
        if constexpr (CS > 1) {
            cluster.sync();
            if (rank == 0 && tid == 0 && p.trace) {
                double s = 0.0;
                for (int q = 0; q < CS; ++q) {
                    const float *rq = cluster.map_shared_rank(red, q);
                    for (int i = 0; i < RB; ++i) s += rq[i];
                }
                p.trace[(size_t)net * p.epochs + e] = s / (double)n;
            }
            cluster.sync();
        } else {
            __syncthreads();
            if (tid == 0 && p.trace) {
                double s = 0.0;
                for (int i = 0; i < kBatchRows; ++i) s += red[i];
                p.trace[(size_t)net * p.epochs + e] = s / (double)n;
            }
        }
    }
    NOMA_PHASE(5)
    if (clk_on)
        for (int i = 0; i < 6; ++i) p.clocks[i] = clk_acc[i];
#undef NOMA_PHASE
    // ---- write the trained parameters back in FusedPlan layout -------------
    if (CS > 1 && rank != 0) return;  // every CTA of the cluster holds the same weights
    float *po = p.plans + (size_t)net * g.plan_total;
    for (int l = 1; l <= N; ++l) {
        const int rowsl = g.dims[l], cols = g.dims[l - 1];
        for (int i = tid; i < rowsl * cols; i += kTrainThreads) {
            const int j = i / cols, c = i % cols;
            po[g.plan_w[l] + j * g.plan_pad[l - 1] + c] = PS[g.pw[l] + j * g.sw[l] + c];
        }
        for (int j = tid; j < rowsl; j += kTrainThreads) po[g.plan_b[l] + j] = PS[g.pb[l] + j];
    }
    for (int j = tid; j < g.dims[N]; j += kTrainThreads) po[g.plan_f + j] = PS[g.pf + j];
}

// host: carve shared memory, pick the moment-slot instantiation, launch.
int train_thr_launch(TrainParams &p, cudaStream_t st, size_t smem, int mom_smem, int need);

// Adam bias-correction constants of every step, FP64 pow as hybrid_nn.cpp:133-135:
// one FP64 pow pair per step in the training kernel sat on the minibatch
// gather's barrier (a long dependent FP64 chain on one thread)
int adam_table_launch(double lr, double b1, double b2, int total, float *t, cudaStream_t st);

__global__ void adam_table_kernel(double lr, double b1, double b2, int total, float *t) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < total) {
        const double c1 = 1.0 - pow(b1, (double)(i + 1));
        const double c2 = 1.0 - pow(b2, (double)(i + 1));
        t[2 * i] = (float)(lr / c1);
        t[2 * i + 1] = (float)(1.0 / c2);
    }
}

int adam_table_launch(double lr, double b1, double b2, int total, float *t, cudaStream_t st) {
    if (total <= 0) return NOMA_OK;
    adam_table_kernel<<<(total + 255) / 256, 256, 0, st>>>(lr, b1, b2, total, t);
    return cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;
}

int train_launch(TrainParams &p, cudaStream_t st) {
    const NetGeom &g = p.g;
    for (int l = 0; l < g.nd; ++l)
        if (g.dims[l] > NOMA_MAX_WIDTH) return NOMA_ERR_UNSUPPORTED;
    if (p.batch < 1 || p.batch > kBatchRows) return NOMA_ERR_UNSUPPORTED;
    int off = 0;
    p.off_x = off;
    off += g.fp[0] * kSR;
    for (int l = 1; l < g.nd; ++l) {
        p.off_a[l] = off;
        off += g.fp[l] * kSR;
    }
    p.off_ps = off;
    off += pad_to(g.ptotal, 4);
    p.gs_stride = pad_to(g.ptotal, 4);
    p.off_gs = off;
    // Prefer (a) two split-K gradient partials and (b) Adam moments in shared
    // memory (frees ~2*ptotal/256 registers per thread for the FFMA2 tiles'
    // scheduling); drop (b) then (a) until the carve-up fits 227 KB.
    const int base_rest = off + kBatchRows * 3 + (g.fp[g.nd - 1] / 16) * kBatchRows + 8;
    auto fits = [&](int splits, int mom) {
        return (size_t)(base_rest + (splits + 2 * mom) * p.gs_stride) * sizeof(float) <= 227 * 1024;
    };
    int mom_smem = 1;
    p.gsplit = kMaxSplit;
    if (!fits(p.gsplit, mom_smem)) p.gsplit = 1;
    if (!fits(p.gsplit, mom_smem)) {
        mom_smem = 0;
        p.gsplit = fits(kMaxSplit, 0) ? kMaxSplit : 1;
    }
    off += p.gsplit * p.gs_stride;
    p.off_mom = off;
    off += 2 * mom_smem * p.gs_stride;
    p.off_r0b = off;
    off += kBatchRows;
    p.off_dy = off;
    off += kBatchRows;
    p.off_red = off;
    off += kBatchRows;
    p.off_yp = off;
    off += (g.fp[g.nd - 1] / 16) * kBatchRows;
    p.off_misc = off;
    off += 8;
    p.off_end = off;
    const size_t smem = (size_t)off * sizeof(float);
    if (smem > 227 * 1024) return NOMA_ERR_UNSUPPORTED;
    const int need = (g.ptotal + 511) / 512;
#define NOMA_TRAIN_LAUNCH(NT, NS, MB)                                                           \
    {                                                                                           \
        cudaFuncSetAttribute(train_kernel<NT, NS, MB, 1>,                                       \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);           \
        p.mode = NT == 256 ? 2 : 1;                                                             \
        train_kernel<NT, NS, MB, 1><<<p.n_nets, NT, smem, st>>>(p);                             \
        return cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;                     \
    }
    // latency mode (few nets, e.g. one slot): a neuron-split cluster per net
    // (k_train_lat.cu); NOMA_LAT_CLUSTER=1 disables it for A/B runs.
    {
        int sms_l = 148, dev_l = 0;
        cudaGetDevice(&dev_l);
        cudaDeviceGetAttribute(&sms_l, cudaDevAttrMultiProcessorCount, dev_l);
        if (p.n_nets * 2 <= sms_l || std::getenv("NOMA_LAT_CLUSTER")) {
            if (train_lat_launch(p, st) == NOMA_OK) return NOMA_OK;
        }
    }
    // throughput kernels: per-step Adam constants precomputed once per launch
    // (unless the caller already did, off the critical path)
    const float *given = p.atab;
    float *tab = nullptr;
    const int total = p.epochs * ((p.rows + p.batch - 1) / p.batch);
    if (given) {
    } else if (total > 0 && cudaMallocAsync(&tab, 2 * (size_t)total * sizeof(float), st) == cudaSuccess) {
        adam_table_kernel<<<(total + 255) / 256, 256, 0, st>>>(p.lr_d, p.b1d, p.b2d, total, tab);
        if (cudaGetLastError() == cudaSuccess) p.atab = tab;
    } else {
        cudaGetLastError();
        tab = nullptr;
    }
    const int r = train_thr_launch(p, st, smem, mom_smem, need);
    if (tab) cudaFreeAsync(tab, st);
    p.atab = given;
    return r;
}

// the throughput kernels (row-split cluster or one CTA per net)
int train_thr_launch(TrainParams &p, cudaStream_t st, size_t smem, int mom_smem, int need) {
    // one hidden layer of 64 (C1, C5): 4-warp CTAs, several nets per SM
    if (train_w4_fits(p)) return train_w4_launch(p, st);
    // one hidden layer of 64 on a 128-wide input (C4): 8-warp CTAs
    if (train_w8_fits(p)) return train_w8_launch(p, st);
    // two hidden layers of 64 on a 32/64-wide input (C2): 8-warp CTAs
    if (train_l2_fits(p)) return train_l2_launch(p, st);
    // row-split cluster: fewer nets than SMs -> a cluster of CS CTAs per net
    int sms = 148;
    {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    int cs = !mom_smem ? 1 : p.n_nets * 4 <= sms ? 4 : p.n_nets * 2 <= sms ? 2 : 1;
    if (const char *force = std::getenv("NOMA_TRAIN_CLUSTER"))  // A/B testing: 1, 2 or 4
        cs = mom_smem && (std::atoi(force) == 2 || std::atoi(force) == 4) ? std::atoi(force) : 1;
    if (cs > 1) {
        auto launch = [&](auto kern) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(p.n_nets * cs);
            cfg.blockDim = dim3(512);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = cs;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            return cudaLaunchKernelEx(&cfg, kern, p) == cudaSuccess;
        };
        const bool ok = cs == 4 ? launch(train_kernel<512, 0, 1, 4>) : launch(train_kernel<512, 0, 1, 2>);
        if (ok) {
            p.mode = 10 + cs;
            return NOMA_OK;
        }
        cudaGetLastError();  // cluster launch refused: fall through to one CTA per net
    }
    // small nets: two 8-warp CTAs (two nets) per SM; else one 16-warp CTA
    // (the 2-per-SM shape only pays when there are more nets than SMs)
    if (mom_smem && smem <= 112 * 1024 && p.n_nets > 148) NOMA_TRAIN_LAUNCH(256, 0, 2)
    if (mom_smem) NOMA_TRAIN_LAUNCH(512, 0, 1)
    if (need <= 8) NOMA_TRAIN_LAUNCH(512, 8, 1)
    if (need <= 16) NOMA_TRAIN_LAUNCH(512, 16, 1)
    if (need <= 24) NOMA_TRAIN_LAUNCH(512, 24, 1)
    if (need <= 32) NOMA_TRAIN_LAUNCH(512, 32, 1)
#undef NOMA_TRAIN_LAUNCH
    return NOMA_ERR_UNSUPPORTED;
}

}  // namespace noma_dev
