// Latency-mode pilot training on sm_100a: hybrid_nn::train (hybrid_nn.cpp:
// 158-195) with loss_and_grad (:84-114) and adam_step (:118-144) for FEW user
// networks (a single slot), one thread-block CLUSTER of CS CTAs per network.
//
// Decomposition: neuron split.  CTA `rank` owns hidden neurons
// [rank*J_l, (rank+1)*J_l) of every layer l (J_l = L_l / CS): their weight
// rows, biases, final-layer weights and Adam moments live in its shared
// memory for the whole training, and it alone updates them -- no gradient
// all-reduce and no weight broadcast.  What crosses the cluster per step:
//   * the final-layer partial outputs yp[r] = sum_{j own} w_j a_N[j][r]
//     (128 floats per CTA, all-to-all) -- the only exchange for one hidden
//     layer (C1);
//   * with N >= 2 hidden layers, the all-gather of a_l (l < N) in the forward
//     pass and the reduce-scatter of dA_l = W_{l+1}^T dZ_{l+1} in the backward
//     -- except in local-dA mode (C2: two layers of 64, 16 CTAs of 8 warps),
//     where the ReLU masks of a_2 travel with the final-layer partials and
//     every owner sends its updated W_2 rows / final weights a step ahead, so
//     each CTA forms dA_1 of its own neurons without a reduce-scatter.
// Exchanges use st.async into the peers' shared memory with mbarrier
// complete_tx byte counting (no cluster-wide barrier per step).  Each CTA sums
// the CS partials in rank order, so every CTA sees the same yhat bit for bit
// and the result is deterministic run to run (test_hybrid_nn.cpp:290-311).
//
// Minibatch input: the IQ-widened rows (iq_transform.cpp:17-20) are gathered
// from the L2-resident FP32 design through the per-epoch permutation
// (hybrid_nn.cpp:176-187) with a two-stage register prefetch (indices two
// steps ahead, rows one step ahead) into a double-buffered feature-major tile.
//
// The frozen linear branch enters through r0 = y - X w0 (FP64, LLS kernel), as
// in the throughput kernel (k_train.cu).
#include <math.h>

#include <cstdlib>
#include <type_traits>

#include "kernels.cuh"
#include "tiles.cuh"

namespace noma_dev {

namespace {


__device__ __forceinline__ uint32_t s2u(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t cl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
// one local arrival + `bytes` of expected remote transactions for the phase
__device__ __forceinline__ void mbar_arm(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// Acquire at CTA scope: the awaited bytes are st.async / bulk-copy writes
// into THIS CTA's shared memory, completed on this CTA's mbarrier (the same
// contract as TMA loads).  A cluster-scope acquire would add an L1
// invalidate-all (CCTL.IVALL) after every wait.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "NOMA_MBW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra NOMA_MBW_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// 16 bytes into a (possibly remote) CTA's shared memory; completes `bytes`
// on that CTA's mbarrier.
__device__ __forceinline__ void st_async4(uint32_t raddr, float4 v, uint32_t rbar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(raddr),
        "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(rbar)
        : "memory");
}

__device__ __forceinline__ void ffma2(f2_t &d, f2_t a, f2_t b) { f2_fma(d, a, b); }

// Bulk async copy of `bytes` (multiple of 16) from this CTA's shared memory to
// a (possibly remote) CTA's shared memory, completing on that CTA's mbarrier.
// The issuing thread must have ordered the source writes (barrier) and made
// them visible to the async proxy (fence_proxy_async) first.
__device__ __forceinline__ void bulk_s2s(uint32_t rdst, uint32_t src, uint32_t bytes, uint32_t rbar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(rdst),
        "r"(src), "r"(bytes), "r"(rbar)
        : "memory");
}
// Bulk async copy global -> the same shared-memory offset of every CTA in
// `mask`, completing on each one's mbarrier at `mbar`'s offset (multicast).
__device__ __forceinline__ void bulk_g2s_mc(uint32_t dst, const void *src, uint32_t bytes, uint32_t mbar,
                                            uint16_t mask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(mbar), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
// Bulk async copy global -> this CTA's shared memory, completing on `mbar`.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(mbar)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// Bulk prefetch of `bytes` (multiple of 16) of global memory into L2.
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

}  // namespace

namespace {

template <int NV>
__device__ __forceinline__ void sts_n(float *p, const float *v) {
    if constexpr (NV == 4) *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
    else if constexpr (NV == 2) *reinterpret_cast<float2 *>(p) = make_float2(v[0], v[1]);
    else *p = v[0];
}

// In-register reduce-scatter of V values (v[0..V)) over a group of LANES
// lanes spaced STR apart (xor offsets (LANES/2) STR .. STR).  Halving rounds
// split the value range on the group-index bits from the top; once one value
// is left the remaining rounds are xor sums.  Afterwards v[0 .. max(1,
// V/LANES)) hold the lane's values: block g of V/LANES values if V >= LANES,
// else the full sum of value index g >> log2(LANES/V), replicated on LANES/V
// lanes (g = (lane / STR) & (LANES-1)).  Fixed summation tree: deterministic.
template <int N, int V, int LANES, int STR = 1>
__device__ __forceinline__ void reduce_scatter(float (&v)[N], int lane) {
    if constexpr (LANES > 1) {
        constexpr int O = LANES / 2;
        if constexpr (V > 1) {
            const bool h = lane & (O * STR);
#pragma unroll
            for (int i = 0; i < V / 2; ++i) {
                const float snd = h ? v[i] : v[i + V / 2];
                const float keep = h ? v[i + V / 2] : v[i];
                v[i] = keep + __shfl_xor_sync(0xffffffffu, snd, O * STR);
            }
            reduce_scatter<N, V / 2, O, STR>(v, lane);
        } else {
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], O * STR);
            reduce_scatter<N, 1, O, STR>(v, lane);
        }
    }
}

// reduce_scatter plus a full xor all-reduce of one more value x at the same
// rounds: x costs no extra dependent shuffle rounds (the bias / final-weight
// gradients ride along with the weight-gradient reduction).
template <int N, int V, int LANES>
__device__ __forceinline__ void reduce_scatter_x(float (&v)[N], float &x, int lane) {
    if constexpr (LANES > 1) {
        constexpr int O = LANES / 2;
        x += __shfl_xor_sync(0xffffffffu, x, O);
        if constexpr (V > 1) {
            const bool h = lane & O;
#pragma unroll
            for (int i = 0; i < V / 2; ++i) {
                const float snd = h ? v[i] : v[i + V / 2];
                const float keep = h ? v[i + V / 2] : v[i];
                v[i] = keep + __shfl_xor_sync(0xffffffffu, snd, O);
            }
            reduce_scatter_x<N, V / 2, O>(v, x, lane);
        } else {
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], O);
            reduce_scatter_x<N, 1, O>(v, x, lane);
        }
    }
}

constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v / 2); }

// Compile-time loop B, B+S, ... (exclusive E): the body sees an
// integral_constant, so layer-dependent tile shapes are constants.
template <int B, int E, int S, typename F>
__device__ __forceinline__ void static_for(F &&f) {
    if constexpr ((S > 0 && B < E) || (S < 0 && B > E)) {
        f(std::integral_constant<int, B>());
        static_for<B + S, E, S>(f);
    }
}

}  // namespace

constexpr int kLatMaxLayers = 2;    // hidden layers handled by the latency kernel
constexpr int kLatMaxSteps = 4096;  // Adam bias-correction table in shared memory
constexpr int kLatMaxHistEpochs = 128;  // epoch-loss history in shared memory (64 KB)

// Shared-memory carve-up (floats), identical on host and device.  Own
// parameters are double-buffered by step parity: step s reads copy s&1 and
// Adam writes copy (s+1)&1, so the update needs no barrier against readers.
struct LatCarve {
    int cs, jt, N, total, width;
    int sw[NOMA_MAX_DIMS];
    int xt, r0b, yall, dy, red, atab;
    int w[NOMA_MAX_DIMS], b[NOMA_MAX_DIMS], wf, npar;  // copy 0; copy 1 at +npar
    int aN;                                            // own a_N [JT][kSR]
    int aloc[NOMA_MAX_DIMS], af[NOMA_MAX_DIMS], rsb[NOMA_MAX_DIMS];  // l < N
    int rsst;                                          // dA partial staging [H][kSR]
    int mk, wt, wfa, wtbar;                            // local-dA mode (two layers of 64 on 16 CTAs), else -1
    int bars;                                          // mbarriers (8-byte aligned)
    int nbars, end;
    int ehist;                                         // epoch-loss history [epochs][128], or -1
};

// Shapes the latency kernel handles (else the caller falls back): 1-2 hidden
// layers of one width H = cs * jt with jt in {2, 4, 8} (jt >= 4 with two
// layers), input width 2M in {32, 64} (k split over 8 lanes, column tiles
// over at most 16 warps), at most kLatMaxSteps Adam steps.
__host__ __device__ inline bool lat_carve(const NetGeom &g, int cs, int width, int total_steps, int epochs,
                                          LatCarve *c) {
    const int N = g.nd - 1;
    if (N < 1 || N > kLatMaxLayers || cs < 2 || cs > 16) return false;
    if (width != g.dims[0] || (width != 32 && width != 64)) return false;
    if (total_steps > kLatMaxSteps) return false;
    const int H = g.dims[1];
    for (int l = 1; l <= N; ++l)
        if (g.dims[l] != H) return false;
    if (H % cs) return false;
    const int jt = H / cs;
    if (jt != 2 && jt != 4 && jt != 8) return false;
    if (N > 1 && (jt < 4 || H > 64)) return false;
    c->cs = cs;
    c->jt = jt;
    c->N = N;
    c->total = total_steps;
    c->width = width;
    int off = 0;
    c->xt = off;
    off += 2 * width * kSR;
    c->r0b = off;
    off += 2 * kBatchRows;
    c->yall = off;
    off += 2 * cs * kBatchRows;
    c->dy = off;
    off += kBatchRows;
    c->red = off;
    off += kBatchRows;
    c->atab = off;
    off += pad_to(2 * total_steps, 4);
    // per-epoch loss partials of the 128 residual threads, reduced once after
    // training (a serial per-epoch sum on rank 0 held the whole cluster up at
    // every epoch end); long runs keep the per-epoch reduction
    c->ehist = -1;
    if (epochs > 0 && epochs <= kLatMaxHistEpochs) {
        c->ehist = off;
        off += epochs * kBatchRows;
    }
    int np = 0;
    for (int l = 1; l <= N; ++l) {
        c->sw[l] = g.dims[l - 1] + 4;
        c->w[l] = off + np;
        np += jt * c->sw[l];
        c->b[l] = off + np;
        np += pad_to(jt, 4);
    }
    c->wf = off + np;
    np += pad_to(jt, 4);
    c->npar = np;
    off += 2 * np;
    c->aN = off;
    off += jt * kSR;
    for (int l = 1; l < N; ++l) {
        c->aloc[l] = off;
        off += jt * kSR;
        c->af[l] = off;  // double-buffered by step parity
        off += 2 * H * kSR;
        c->rsb[l] = off;
        off += cs * jt * kSR;
    }
    c->rsst = off;
    if (N > 1) off += H * kSR;
    // local-dA mode: ReLU masks of every CTA's a2 [2][cs][jt][4] words, the
    // own layer-1 neurons' columns of W2 [2][H][4] and all final weights [2][H]
    c->mk = c->wt = c->wfa = c->wtbar = -1;
    const bool lda = N == 2 && jt == 4 && cs == 16 && width == 32;  // the 8-warp instance (train_lat_kernel LDA)
    if (lda) {
        c->mk = off;
        off += 2 * cs * 16;
        c->wt = off;
        off += 2 * H * 4;
        c->wfa = off;
        off += 2 * H;
    }
    off = pad_to(off, 2);
    c->bars = off;
    c->nbars = 2 + 2 * (N - 1) + (lda ? 2 : 0) + 2;  // Y[2], AG_l, RS_l, [WT[2]], G[2] (minibatch tiles)
    if (lda) c->wtbar = 2 + 2 * (N - 1);
    off += 2 * c->nbars;
    c->end = off;
    return (size_t)off * sizeof(float) <= 227 * 1024;
}

template <int CS, int JT, int NL, int VW, int NW>
__global__ void __launch_bounds__(NW * 32, 1) train_lat_kernel(TrainParams p, LatCarve c) {
    constexpr int kLT = NW * 32;  // threads per CTA (16 warps, or 8 for one 32-input layer)
    extern __shared__ __align__(16) float sm[];
    constexpr int H = CS * JT;
    const int net = blockIdx.x / CS;
    if (p.status && p.status[net] != NOMA_OK) return;  // uniform over the cluster
    // detection (programmatic dependent launch) may take the idle SMs for its
    // prologue; it waits for this grid before reading the trained plans
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint32_t rank = cl_rank();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const NetGeom &g = p.g;
    const int n = p.rows, d = net / p.K, width = c.width, M = width / 2;
    const bool wid = p.layout == NOMA_LAYOUT_WIDEN_COMPLEX;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + c.bars);
    // barrier indices: Y[0], Y[1], then AG_l = 2 + 2(l-1), RS_l = 3 + 2(l-1)
    // phase cycles (NOMA_PHASE_CLOCKS, block 0 thread 0): 0 forward, 1 its
    // barrier, 2 yp send + gather, 3 yp wait, 4 residual + barrier, 5 backward
    // + Adam, 6 end-of-step barrier, 7 prologue / epilogue.  After a barrier a
    // volatile shared load blocks until the barrier has actually released.
    const bool clk_on = NOMA_PROBE_ON(p.clocks && blockIdx.x == 0 && tid == 0);
    long long clk_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, clk_prev = clk_on ? clock64() : 0;
#ifdef NOMA_PROBES
#define NOMA_LPHASE(I)                                            \
    if (clk_on) {                                                 \
        (void)*reinterpret_cast<volatile float *>(sm + c.dy);     \
        const long long now = clock64();                          \
        clk_acc[I] += now - clk_prev;                             \
        clk_prev = now;                                           \
    }
#else
#define NOMA_LPHASE(I)
#endif
    // per-warp timeline of steps 100-103 (lane 0 of every warp of block 0)
    long long *tl = p.clocks && blockIdx.x == 0 && lane == 0 ? p.clocks + 8 + warp * 16 : nullptr;
#ifdef NOMA_PROBES
#define NOMA_TL(PT)                                                              \
    if (tl && s >= 100 && s < 104) tl[(s - 100) * 256 + (PT)] = clock64();
    // cross-CTA timeline (globaltimer, ns): thread 0 of the first cluster's
    // CTAs at step 101, slots [8 + 1024 + 16 * block + PT]
#define NOMA_GT(PT)                                                                       \
    if (p.clocks && tid == 0 && blockIdx.x < 16 && s == 101) {                            \
        unsigned long long gt_;                                                           \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_));                           \
        p.clocks[8 + 1024 + 16 * blockIdx.x + (PT)] = (long long)gt_;                     \
    }
#else
#define NOMA_TL(PT)
#define NOMA_GT(PT)
#endif

    for (int i = tid; i < c.bars; i += kLT) sm[i] = 0.0f;
    __syncthreads();
    // own parameters (copy 0) from the FusedPlan buffer (fused_inference.cpp:19-42)
    const float *pl = p.plans + (size_t)net * g.plan_total;
#pragma unroll
    for (int l = 1; l <= NL; ++l) {
        const int C = g.dims[l - 1];
        for (int i = tid; i < JT * C; i += kLT) {
            const int j = i / C, k = i - j * C;
            sm[c.w[l] + j * c.sw[l] + k] = pl[g.plan_w[l] + (rank * JT + j) * g.plan_pad[l - 1] + k];
        }
        if (tid < JT) sm[c.b[l] + tid] = pl[g.plan_b[l] + rank * JT + tid];
    }
    if (tid < JT) sm[c.wf + tid] = pl[g.plan_f + rank * JT + tid];
    // Adam bias corrections per step, FP64 pow like hybrid_nn.cpp:133-135
    for (int i = tid; i < c.total; i += kLT) {
        if (p.atab) {  // precomputed beside the LLS (adam_table_kernel, same arithmetic)
            sm[c.atab + 2 * i] = p.atab[2 * i];
            sm[c.atab + 2 * i + 1] = p.atab[2 * i + 1];
        } else {
            const double c1 = 1.0 - pow(p.b1d, (double)(i + 1));
            const double c2 = 1.0 - pow(p.b2d, (double)(i + 1));
            sm[c.atab + 2 * i] = (float)(p.lr_d / c1);
            sm[c.atab + 2 * i + 1] = (float)(1.0 / c2);
        }
    }
    // Local-dA mode (C2: two layers of 64 on 16 CTAs of 8 warps): instead of
    // reduce-scattering dA1 partials (16 x 2 KB per CTA per step), every CTA
    // receives the ReLU masks of all a2 rows with the final-layer partials (64
    // bytes per peer) and keeps W2's columns of its own layer-1 neurons and all
    // final weights current (each owner sends its updated rows after Adam, a
    // whole step ahead of use), and forms dA1 of its own neurons locally.
    constexpr bool LDA = NL == 2 && JT == 4 && NW == 8 && CS == 16;
    constexpr uint32_t ybytes = CS * kBatchRows * 4 + (LDA ? CS * 64 : 0);
    constexpr uint32_t wtbytes = CS * (JT * 16 + 16);
    // all-gather / reduce-scatter move whole [JT][kSR] tiles by bulk copy
    // local-dA mode: the a1 all-gather leaves per warp (kBatchRows columns
    // only, the pad columns of af stay zero from the start)
    const bool WMC = LDA && p.agbuf;  // uniform over the cluster
    const uint32_t agbytes = H * (WMC ? kBatchRows : kSR) * 4;
    constexpr uint32_t rsbytes = CS * JT * kSR * 4;
    if (tid == 0) {
        for (int b = 0; b < c.nbars; ++b) mbar_init(s2u(bars + b), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_arm(s2u(bars + 0), ybytes);
        mbar_arm(s2u(bars + 1), ybytes);
#pragma unroll
        for (int l = 1; l < NL; ++l) {
            mbar_arm(s2u(bars + 2 + 2 * (l - 1)), agbytes);
            mbar_arm(s2u(bars + 3 + 2 * (l - 1)), rsbytes);
        }
        if constexpr (LDA) {
            mbar_arm(s2u(bars + c.wtbar), 0);             // phase 0: step 0 (initial weights)
            mbar_arm(s2u(bars + c.wtbar), wtbytes);       // phase 1: step 2
            mbar_arm(s2u(bars + c.wtbar + 1), wtbytes);   // phase 0: step 1
        }
    }
    if constexpr (LDA) {  // step 0's W2 columns and final weights from the plans
        for (int t = tid; t < H * JT; t += kLT)
            sm[c.wt + t] = pl[g.plan_w[2] + (t / JT) * g.plan_pad[1] + rank * JT + t % JT];
        for (int t = tid; t < H; t += kLT) sm[c.wfa + t] = pl[g.plan_f + t];
    }

    // ---- step schedule: minibatch tiles by bulk copy --------------------------
    // lat_prep_kernel has materialised every step's permuted, IQ-widened,
    // feature-major tile X[W0][kSR] and its r0 column (hybrid_nn.cpp:176-187,
    // iq_transform.cpp:17-20); one thread copies step s+1's tile into the other
    // buffer during step s, completing on barrier G[(s+1)&1].
    constexpr int W0 = 16 * VW;  // input width 2M
    const int spe = (n + p.batch - 1) / p.batch;  // steps per epoch
    const int total = c.total;
    constexpr uint32_t xbytes = W0 * kSR * 4, rbytes = kBatchRows * 4;
    const int gbar0 = c.nbars - 2;
    // L2 prefetch distance (steps); one hidden layer only: a C2 step (~4 us)
    // already covers the fetch (C1 train 803 -> 789 us, C2 +0.4 % with it)
    constexpr int kPfd = NL == 1 ? 3 : 0;
    const float *xsrc = p.xprep + (size_t)net * total * W0 * kSR;
    const float *rsrc = p.r0prep + (size_t)net * total * kBatchRows;
    auto fetch = [&](int step) {  // one thread
        const int b = step & 1;
        const uint32_t gb = s2u(bars + gbar0 + b);
        mbar_arm(gb, xbytes + rbytes);
        bulk_g2s(s2u(sm + c.xt + b * W0 * kSR), xsrc + (size_t)step * W0 * kSR, xbytes, gb);
        bulk_g2s(s2u(sm + c.r0b + b * kBatchRows), rsrc + (size_t)step * kBatchRows, rbytes, gb);
    };
    (void)wid;
    (void)d;
    (void)M;
    __syncthreads();
    if (tid == kLT - 32 && total > 0) {
        fetch(0);  // same issuer as every later fetch
        for (int q = 1; q < kPfd && q < total; ++q) {
            bulk_prefetch_l2(xsrc + (size_t)q * W0 * kSR, xbytes);
            bulk_prefetch_l2(rsrc + (size_t)q * kBatchRows, rbytes);
        }
    }
    cl_sync();  // every CTA's barriers initialised before any st.async lands

    // Adam moments of the parameters this thread updates (registers; fixed
    // thread -> parameter map for the whole training): per layer one weight
    // and one bias-or-final-weight.
    // (up to 2 column tiles per warp when a layer has more tiles than warps)
    float mw[NL + 1][2], vw[NL + 1][2], mb[NL + 1], vb[NL + 1];
#pragma unroll
    for (int l = 0; l <= NL; ++l) mw[l][0] = vw[l][0] = mw[l][1] = vw[l][1] = mb[l] = vb[l] = 0.f;

    // forward thread map: KSF k-split lanes x 32 row quads x NW / KSF neuron
    // groups; after the k reduce-scatter a lane holds FV values (neuron fj,
    // rows 4 frq + fr ..), or -- with fewer values than lanes -- one value on
    // KSF / FVV lanes.  On 8 warps k splits over 4 lanes and the neurons over
    // two groups: one shuffle round less than 8 lanes, at twice the input
    // loads (C1 -1.3 %, C2 -0.9 %; for the first layer the end-of-step
    // preload hides them).  Two layers with 8 lanes and one group (each
    // gathered a1 element read once) measured the same once the dZ1 sum ran
    // on all warps.
    constexpr int KSF = (NW == 8 && JT % 2 == 0) ? 4 : 8;
    constexpr int JPF = JT / (NW / KSF);         // neurons per forward thread
    constexpr int FVV = 4 * JPF;                 // values before the reduce
    constexpr int FV = FVV >= KSF ? FVV / KSF : 1;  // values per lane after it
    // The KSF k lanes of a row quad sit STR = 32 / KSF lanes apart, so the 8
    // lanes of a 16-byte load phase read 8 consecutive row quads of one
    // k-quad: bank groups (4 kc + kk + frq) mod 8 all differ.  (Adjacent k
    // lanes put k-quads kc and kc + 2 in one phase -- bank groups 4 kc mod 8
    // coincide -- a 2-way conflict on every activation load of the forward.)
    constexpr int FSTR = 32 / KSF;
    const int fkq = lane / FSTR, frq = (lane & (FSTR - 1)) | ((warp % KSF) * FSTR), fjh = warp / KSF;
    const int fbase = FVV >= KSF ? fkq * FV : fkq >> (ilog2c(KSF) - ilog2c(FVV));
    const bool fown = FVV >= KSF || (fkq & ((KSF / FVV) - 1)) == 0;
    const int fj = fjh * JPF + (fbase >> 2), fr = fbase & 3;

    float loss_acc = 0.0f;
    int s = 0;
    // The forward's input operands of the next step are loaded at the end of
    // the current one (after its tile's barrier), so their shared-memory
    // latency hides behind the end-of-step barrier instead of heading the
    // forward's chain.
    constexpr int NCI = W0 / 4 / KSF;  // input k-quads per forward lane
    ulonglong2 fx[NCI][4];
    auto load_fx = [&](int step) {
        mbar_wait(s2u(bars + gbar0 + (step & 1)), (uint32_t)((step >> 1) & 1));  // the step's tile
        const float *xt = sm + c.xt + (step & 1) * width * kSR;
#pragma unroll
        for (int ci = 0; ci < NCI; ++ci)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
                fx[ci][kk] = *reinterpret_cast<const ulonglong2 *>(xt + 4 * (fkq + KSF * ci) * kSR + 4 * frq + kk * kSR);
    };
    if (total > 0) load_fx(0);
    // weight-gradient operands of one hidden layer (C1): the input columns and
    // activations are final after the forward's barrier; every warp loads its
    // tile while the final-layer partials cross the cluster
    constexpr int PNCL = W0 / 4;
    constexpr bool kPre = NL == 1 && PNCL <= NW;
    constexpr int PJPB = JT / (PNCL >= NW ? 1 : NW / PNCL);
    // two layers with one input column tile per warp: the first layer's
    // weight-gradient inputs are loaded before the dA reduce-scatter wait
    constexpr bool kPre1 = NL > 1 && W0 / 4 == NW && !LDA;
    ulonglong2 bx[4];
    float4 bz[PJPB];
    NOMA_LPHASE(7)
    for (int e = 0; e < p.epochs; ++e) {
        for (int st = 0; st < spe; ++st, ++s) {
            const int buf = s & 1;
            const int start = st * p.batch, bsz = min(p.batch, n - start);
            const float *XT = sm + c.xt + buf * width * kSR;
            const int po = buf * c.npar, pn = (buf ^ 1) * c.npar;  // param copy: read, write
            NOMA_TL(0)
            NOMA_GT(0)
            // ---- forward (hybrid_nn.cpp:60-72): all JT own neurons x 4 rows per
            // thread, k split over 8 lanes, lane reduce-scatter --------------
static_for<1, NL + 1, 1>([&](auto LC) {
                constexpr int l = decltype(LC)::value;
                const int NC = (l == 1 ? W0 : H) >> 2;
                const float *in = l == 1 ? XT : sm + c.af[l - 1] + buf * H * kSR;
                const float *W = sm + po + c.w[l] + fjh * JPF * c.sw[l];
                const int sw = c.sw[l];
                {
                    f2_t acc[JPF][2];
#pragma unroll
                    for (int j = 0; j < JPF; ++j) acc[j][0] = acc[j][1] = 0ull;
#pragma unroll
                    for (int kc = fkq; kc < NC; kc += KSF) {
                        const float *ip = in + 4 * kc * kSR + 4 * frq;
                        ulonglong2 x[4];
                        if constexpr (l == 1) {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk) x[kk] = fx[kc / KSF][kk];
                        } else {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk) x[kk] = *reinterpret_cast<const ulonglong2 *>(ip + kk * kSR);
                        }
#pragma unroll
                        for (int j = 0; j < JPF; ++j) {
                            const float4 w4 = *reinterpret_cast<const float4 *>(W + j * sw + 4 * kc);
                            const float wk[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk) {
                                const f2_t wb = f2_bcast(wk[kk]);
                                ffma2(acc[j][0], wb, x[kk].x);
                                ffma2(acc[j][1], wb, x[kk].y);
                            }
                        }
                    }
                    float v[FVV];
#pragma unroll
                    for (int j = 0; j < JPF; ++j) {
                        const float2 a = f2_unpack(acc[j][0]), b = f2_unpack(acc[j][1]);
                        v[4 * j] = a.x;
                        v[4 * j + 1] = a.y;
                        v[4 * j + 2] = b.x;
                        v[4 * j + 3] = b.y;
                    }
                    reduce_scatter<FVV, FVV, KSF, FSTR>(v, lane);
                    const float bj = sm[po + c.b[l] + fj];
#pragma unroll
                    for (int i = 0; i < FV; ++i) v[i] = fmaxf(v[i] + bj, 0.f);
                    const int r = 4 * frq + fr;
                    if (fown) sts_n<FV>((l == NL ? sm + c.aN : sm + c.aloc[l]) + fj * kSR + r, v);
                    if (l < NL && p.agbuf) {  // staged in global for the multicast all-gather
                        float *gt = p.agbuf + ((size_t)net * 2 + buf) * H * kSR + rank * JT * kSR;
                        if (fown) sts_n<FV>(gt + fj * kSR + r, v);
                        if (!WMC && tid < JT * (kSR - kBatchRows))  // pad columns stay zero
                            gt[(tid / (kSR - kBatchRows)) * kSR + kBatchRows + tid % (kSR - kBatchRows)] = 0.0f;
                        fence_proxy_async_global();
                        if (WMC) {
                            // this warp's 32 rows of its two neurons leave as soon
                            // as they are written: one multicast per neuron row
                            __syncwarp();
                            if (lane < JPF) {
                                const int nj = fjh * JPF + lane, c0 = 32 * (warp % KSF);
                                bulk_g2s_mc(s2u(sm + c.af[l] + (buf * H + rank * JT + nj) * kSR + c0),
                                            gt + nj * kSR + c0, 128, s2u(bars + 2 + 2 * (l - 1)),
                                            (uint16_t)((1u << CS) - 1));
                            }
                        }
                    }
                }
                if (l < NL) {
                    // all-gather a_l: the own [JT][kSR] tile to every CTA (incl.
                    // this one) by bulk copy, rows rank*JT.. of af_l[s&1].  The
                    // source is rewritten only at step s+1, after every copy
                    // of step s has landed (peers' RS of step s waits on it);
                    // af is double-buffered because the RS copies are issued
                    // before this CTA's last read of af (the weight gradient).
                    const uint32_t lb = s2u(bars + 2 + 2 * (l - 1));
                    NOMA_TL(10)
                    NOMA_GT(1)
                    if (!WMC) __syncthreads();
                    if (WMC) {
                    } else if (p.agbuf) {
                        // one multicast copy from the global staging tile into
                        // every CTA's af slot (the SM's outbound smem -> peer
                        // copies ran at ~16 B/clk: 34 KB per step)
                        if (tid == 0)
                            bulk_g2s_mc(s2u(sm + c.af[l] + (buf * H + rank * JT) * kSR),
                                        p.agbuf + ((size_t)net * 2 + buf) * H * kSR + rank * JT * kSR,
                                        JT * kSR * 4, lb, (uint16_t)((1u << CS) - 1));
                    } else if (tid < CS) {  // destination order rotated by rank: each CTA's
                                            // copies do not all queue for the same peer first
                        const uint32_t dst = (rank + tid) % CS;
                        fence_proxy_async();
                        bulk_s2s(mapa(s2u(sm + c.af[l] + (buf * H + rank * JT) * kSR), dst), s2u(sm + c.aloc[l]),
                                 JT * kSR * 4, mapa(lb, dst));
                    }
                    mbar_wait(lb, (uint32_t)(s & 1));
                    NOMA_TL(11)
                    NOMA_GT(2)
                    // re-arm for step s+1 (its bytes cannot land before every
                    // CTA has finished step s)
                    if (tid == 0) mbar_arm(lb, agbytes);
                }
            });
            NOMA_LPHASE(0)
            NOMA_TL(1)
            NOMA_GT(3)
            __syncthreads();
            NOMA_LPHASE(1)
            NOMA_TL(2)
            // ---- final-layer partials yp (hybrid_nn.cpp:81): kYW warps send ---
            const uint32_t ybar = s2u(bars + buf);
            // two layers: every warp computes the (cheap) partial and sends to
            // CS / NW peers (C2 -16 us); one layer: warps 0-1, 8 peers each
            // (4 warps: +3 us, all 8: +42 us; the other warps preload the
            // weight-gradient operands meanwhile)
            constexpr int kYW = NL > 1 ? (NW < CS ? NW : CS) : 2;
            if (warp < kYW) {
                const int r0 = 4 * lane;
                const float *aN = sm + c.aN;
                const float *wf = sm + po + c.wf;
                float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int j = 0; j < JT; ++j) {
                    const float4 a = *reinterpret_cast<const float4 *>(aN + j * kSR + r0);
                    const float f = wf[j];
                    y.x = fmaf(f, a.x, y.x);
                    y.y = fmaf(f, a.y, y.y);
                    y.z = fmaf(f, a.z, y.z);
                    y.w = fmaf(f, a.w, y.w);
                }
                const uint32_t la = s2u(sm + c.yall + (buf * CS + rank) * kBatchRows + r0);
#pragma unroll
                for (int q = warp; q < CS; q += kYW) {
                    // two layers: destinations rotated by rank (as the bulk
                    // exchanges); one layer: in order (rotated measured +2 %)
                    const uint32_t dst = NL > 1 ? (rank + q) % CS : q;
                    st_async4(mapa(la, dst), y, mapa(ybar, dst));
                }
                if constexpr (LDA) {
                    // ReLU mask of the own a2: word 4 j + k = rows 32 k .. 32 k + 31 of
                    // neuron j; lanes 0-3 send 16 bytes each to this warp's peers
                    uint32_t mw = 0;
#pragma unroll
                    for (int j = 0; j < JT; ++j)
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const uint32_t bt = __ballot_sync(0xffffffffu, aN[j * kSR + 32 * k + lane] > 0.f);
                            if (lane == 4 * j + k) mw = bt;
                        }
                    const uint32_t m0 = __shfl_sync(0xffffffffu, mw, (4 * lane) & 31),
                                   m1 = __shfl_sync(0xffffffffu, mw, (4 * lane + 1) & 31),
                                   m2 = __shfl_sync(0xffffffffu, mw, (4 * lane + 2) & 31),
                                   m3 = __shfl_sync(0xffffffffu, mw, (4 * lane + 3) & 31);
                    if (lane < 4) {
                        const uint32_t ma = s2u(sm + c.mk + (buf * CS + rank) * 16 + 4 * lane);
                        const float4 mv = make_float4(__uint_as_float(m0), __uint_as_float(m1), __uint_as_float(m2),
                                                      __uint_as_float(m3));
#pragma unroll
                        for (int q = warp; q < CS; q += kYW) {
                            const uint32_t dst = (rank + q) % CS;
                            st_async4(mapa(ma, dst), mv, mapa(ybar, dst));
                        }
                    }
                }
            }
            NOMA_TL(3)
            NOMA_GT(4)
            // ---- next step's minibatch tile (bulk copy, one thread off the
            // critical warps; XT[buf^1] was last read in step s-1) ------------
            if (tid == kLT - 32 && s + 1 < total) fetch(s + 1);
            // the tile kPfd steps ahead into L2: the bulk copy of step s+1's
            // tile otherwise starts from HBM (the prepared tiles of a C1 slot
            // are 56 MB) and was still landing when step s ended
            if (kPfd > 0 && tid == kLT - 32 && s + kPfd < total) {
                bulk_prefetch_l2(xsrc + (size_t)(s + kPfd) * W0 * kSR, xbytes);
                bulk_prefetch_l2(rsrc + (size_t)(s + kPfd) * kBatchRows, rbytes);
            }
            if constexpr (kPre) {
                const int ct = warp % PNCL, jg = warp / PNCL, r = 4 * lane;
#pragma unroll
                for (int q = 0; q < 4; ++q) bx[q] = *reinterpret_cast<const ulonglong2 *>(XT + (4 * ct + q) * kSR + r);
#pragma unroll
                for (int j = 0; j < PJPB; ++j) bz[j] = *reinterpret_cast<const float4 *>(sm + c.aN + (jg * PJPB + j) * kSR + r);
            }
            NOMA_LPHASE(2)
            NOMA_TL(4)
            // ---- residual a_N w - r0, dy = 2 r / B (hybrid_nn.cpp:94-98): warps
            // 0-3, one row per lane, partials summed in rank order ------------
            if (warp < 4) {
                mbar_wait(ybar, (uint32_t)((s >> 1) & 1));
                NOMA_LPHASE(3)
                NOMA_TL(5)
                NOMA_GT(5)
                const int r = tid;  // 0..127
                const float *ya = sm + c.yall + buf * CS * kBatchRows + r;
                float yq[CS];
#pragma unroll
                for (int q = 0; q < CS; ++q) yq[q] = ya[q * kBatchRows];
                // fixed pairwise tree, identical on every CTA of the cluster
                // (each computes the residual of all rows; C1 -10 us vs a chain)
#pragma unroll
                for (int w = 1; w < CS; w *= 2)
#pragma unroll
                    for (int q = 0; q + w < CS; q += 2 * w) yq[q] += yq[q + w];
                const float yh = yq[0];
                const float res = r < bsz ? yh - sm[c.r0b + buf * kBatchRows + r] : 0.0f;
                sm[c.dy + r] = (2.0f / (float)bsz) * res;
                loss_acc = fmaf(res, res, loss_acc);
            }
            NOMA_TL(6)
            __syncthreads();
            if (tid == 0) mbar_arm(ybar, ybytes);  // phase for step s+2
            NOMA_LPHASE(4)
            NOMA_TL(7)
            // ---- backward (hybrid_nn.cpp:99-112) fused with Adam (:118-144) ---
            const float lrc = sm[c.atab + 2 * s], ic2 = sm[c.atab + 2 * s + 1];
static_for<NL, 0, -1>([&](auto LC) {
                constexpr int l = decltype(LC)::value;
                const bool top = l == NL;
                const float *zsrc = top ? sm + c.aN : sm + c.aloc[l];  // a_N, or dZ_l in place
                const float *dyp = sm + c.dy, *wfp = sm + po + c.wf;
                const float *in = l == 1 ? XT : sm + c.af[l - 1] + buf * H * kSR;
                const int sw = c.sw[l];
                if constexpr (LDA && l == 2) {
                    // dA1[j][r] = sum_i W2[i][own j] dZ2[i][r] (:111) for the own
                    // layer-1 neurons, dZ2[i][r] = mask_i[r] dy[r] wf[i] (:102-107):
                    // lane = 8 i-splits x 4 row quads, warps over row quads; the
                    // 8-lane reduce-scatter leaves two rows of one neuron per lane
                    const int b = s & 1;
                    if (s > 0) mbar_wait(s2u(bars + c.wtbar + b), (uint32_t)((s >> 1) & 1));
                    const int ks = lane & 7, rq = (lane >> 3) + 4 * warp, r = 4 * rq;
                    const float4 dy4 = *reinterpret_cast<const float4 *>(dyp + r);
                    const uint32_t *mk = reinterpret_cast<const uint32_t *>(sm + c.mk) + buf * CS * 16 + (rq >> 3);
                    const int sh = 4 * (rq & 7);
                    f2_t acc[JT][2];
#pragma unroll
                    for (int j = 0; j < JT; ++j) acc[j][0] = acc[j][1] = 0ull;
#pragma unroll
                    for (int ii = 0; ii < H / 8; ++ii) {
                        const int i = 8 * ii + ks;
                        const float4 w = *reinterpret_cast<const float4 *>(sm + c.wt + (b * H + i) * 4);
                        const float f = sm[c.wfa + b * H + i];
                        const uint32_t bits = mk[(i >> 2) * 16 + (i & 3) * 4] >> sh;
                        const f2_t za = f2_pack(bits & 1u ? dy4.x * f : 0.f, bits & 2u ? dy4.y * f : 0.f);
                        const f2_t zb = f2_pack(bits & 4u ? dy4.z * f : 0.f, bits & 8u ? dy4.w * f : 0.f);
                        const float wc[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                        for (int j = 0; j < JT; ++j) {
                            const f2_t wj = f2_bcast(wc[j]);
                            ffma2(acc[j][0], wj, za);
                            ffma2(acc[j][1], wj, zb);
                        }
                    }
                    float v[4 * JT];
#pragma unroll
                    for (int j = 0; j < JT; ++j) {
                        const float2 u = f2_unpack(acc[j][0]), t2 = f2_unpack(acc[j][1]);
                        v[4 * j] = u.x;
                        v[4 * j + 1] = u.y;
                        v[4 * j + 2] = t2.x;
                        v[4 * j + 3] = t2.y;
                    }
                    reduce_scatter<4 * JT, 4 * JT, 8>(v, lane);
                    // dZ1 own = (a1 > 0) dA1, in place
                    float2 *ap = reinterpret_cast<float2 *>(sm + c.aloc[1] + (ks >> 1) * kSR + r + 2 * (ks & 1));
                    const float2 a = *ap;
                    *ap = make_float2(a.x > 0.f ? v[0] : 0.f, a.y > 0.f ? v[1] : 0.f);
                }
                if (l > 1 && !LDA)
                for (int tt = tid; tt < (H / 4) * 32; tt += kLT) {
                    // dA_{l-1} partial = sum_{j own} W_l[j][c] dZ_l[j][r] (:111) for
                    // every c (4 c x 4 r per thread), sent to the owner of c.
                    const float *W = sm + po + c.w[l];
                    const uint32_t rb = s2u(bars + 3 + 2 * (l - 2));
                    // JT == 4: column quad = one peer's tile; quads rotated by rank
                    // so the CTAs' early copies go to different peers
                    const int cq = JT == 4 ? ((tt >> 5) + (int)rank) % (H / 4) : tt >> 5;
                    const int r = 4 * lane, cc = 4 * cq;
                    f2_t acc[4][2];
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = 0ull;
                    float4 y4 = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (top) y4 = *reinterpret_cast<const float4 *>(dyp + r);
#pragma unroll
                    for (int j = 0; j < JT; ++j) {
                        const float4 w4 = *reinterpret_cast<const float4 *>(W + j * sw + cc);
                        float4 z = *reinterpret_cast<const float4 *>(zsrc + j * kSR + r);
                        if (top) {
                            const float f = wfp[j];
                            z = make_float4(z.x > 0.f ? y4.x * f : 0.f, z.y > 0.f ? y4.y * f : 0.f,
                                            z.z > 0.f ? y4.z * f : 0.f, z.w > 0.f ? y4.w * f : 0.f);
                        }
                        const f2_t za = f2_pack(z.x, z.y), zb = f2_pack(z.z, z.w);
                        const float wc[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const f2_t wq = f2_bcast(wc[q]);
                            ffma2(acc[q][0], wq, za);
                            ffma2(acc[q][1], wq, zb);
                        }
                    }
                    (void)rb;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float2 u = f2_unpack(acc[q][0]), v = f2_unpack(acc[q][1]);
                        *reinterpret_cast<float4 *>(sm + c.rsst + (cc + q) * kSR + r) = make_float4(u.x, u.y, v.x, v.y);
                    }
                    if constexpr (JT == 4) {
                        // reduce-scatter as soon as this warp's tile is done:
                        // rows [cq*JT, (cq+1)*JT) of the partial to CTA cq's
                        // slot `rank` (single-buffered: rewritten at step s+1
                        // only after every peer has consumed step s)
                        fence_proxy_async();
                        __syncwarp();
                        if (lane == 0)
                            bulk_s2s(mapa(s2u(sm + c.rsb[l - 1] + rank * JT * kSR), cq),
                                     s2u(sm + c.rsst + cq * JT * kSR), JT * kSR * 4, mapa(rb, cq));
                    }
                }
                if (l > 1) {
                    // reduce-scatter: rows [q*JT, (q+1)*JT) of the partial to CTA
                    // q's slot `rank` (single-buffered: rewritten at step s+1 only
                    // after every peer has consumed step s, see the Y exchange)
                    const uint32_t rb = s2u(bars + 3 + 2 * (l - 2));
                    if constexpr (JT != 4) {
                        __syncthreads();
                        if (tid < CS) {
                            const uint32_t dst = (rank + tid) % CS;
                            fence_proxy_async();
                            bulk_s2s(mapa(s2u(sm + c.rsb[l - 1] + rank * JT * kSR), dst),
                                     s2u(sm + c.rsst + dst * JT * kSR), JT * kSR * 4, mapa(rb, dst));
                        }
                    }
                    (void)rb;
                    NOMA_TL(12)
                }
                // weight gradient dZ^T A (:109), bias colsum (:110), final a_N^T dy
                // (:99): warp ct owns column tile 4ct..4ct+3 for all JT neurons,
                // lane = row quad; lane reduce-scatter, then Adam in registers.
                constexpr int NCL = (l == 1 ? W0 : H) / 4;
                constexpr int TPW = NCL > NW ? NCL / NW : 1;  // column tiles per warp
                static_assert(TPW <= 2 && (NCL <= NW || NCL % NW == 0), "tile map");
                // Two column tiles per warp (C2's second layer on 8 warps): both
                // tiles' 2 x 4 JT sums go through ONE 32-value reduce-scatter (5
                // dependent shuffle rounds instead of 2 x 5, and every lane then
                // owns one weight), the dZ operands are loaded once for both, and
                // the bias / final-weight sums ride along as in XSPREAD.
                constexpr int NXP = (l == NL ? 2 : 1) * JT;
                constexpr bool PAIR = TPW == 2 && 8 * JT == 32 && NXP <= NW;
                if constexpr (PAIR) {
                    const int r = 4 * lane;
                    f2_t acc[2][JT][4], sb[JT], sf[JT];
#pragma unroll
                    for (int j = 0; j < JT; ++j) {
                        sb[j] = sf[j] = 0ull;
#pragma unroll
                        for (int q = 0; q < 4; ++q) acc[0][j][q] = acc[1][j][q] = 0ull;
                    }
                    ulonglong2 x[2][4];
#pragma unroll
                    for (int tw = 0; tw < 2; ++tw)
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            x[tw][q] = *reinterpret_cast<const ulonglong2 *>(in + (4 * (warp + NW * tw) + q) * kSR + r);
                    float4 y4 = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (top) y4 = *reinterpret_cast<const float4 *>(dyp + r);
                    const f2_t one = f2_bcast(1.0f);
#pragma unroll
                    for (int j = 0; j < JT; ++j) {
                        float4 z = *reinterpret_cast<const float4 *>(zsrc + j * kSR + r);
                        if (top) {  // dZ_N = (a_N > 0) dy w_j on the fly (:102-107)
                            ffma2(sf[j], f2_pack(z.x, z.y), f2_pack(y4.x, y4.y));
                            ffma2(sf[j], f2_pack(z.z, z.w), f2_pack(y4.z, y4.w));
                            const float f = wfp[j];
                            z = make_float4(z.x > 0.f ? y4.x * f : 0.f, z.y > 0.f ? y4.y * f : 0.f,
                                            z.z > 0.f ? y4.z * f : 0.f, z.w > 0.f ? y4.w * f : 0.f);
                        }
                        const f2_t za = f2_pack(z.x, z.y), zb = f2_pack(z.z, z.w);
                        ffma2(sb[j], za, one);
                        ffma2(sb[j], zb, one);
#pragma unroll
                        for (int tw = 0; tw < 2; ++tw)
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                ffma2(acc[tw][j][q], za, x[tw][q].x);
                                ffma2(acc[tw][j][q], zb, x[tw][q].y);
                            }
                    }
                    float gv[32];
#pragma unroll
                    for (int tw = 0; tw < 2; ++tw)
#pragma unroll
                        for (int j = 0; j < JT; ++j)
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const float2 h = f2_unpack(acc[tw][j][q]);
                                gv[16 * tw + 4 * j + q] = h.x + h.y;
                            }
                    float ex = 0.f;  // warp w < JT: bias w; JT <= w < 2 JT: final weight w - JT
#pragma unroll
                    for (int j = 0; j < JT; ++j) {
                        if (warp == j) {
                            const float2 h = f2_unpack(sb[j]);
                            ex = h.x + h.y;
                        }
                        if (top && warp == JT + j) {
                            const float2 h = f2_unpack(sf[j]);
                            ex = h.x + h.y;
                        }
                    }
                    reduce_scatter_x<32, 32, 32>(gv, ex, lane);
                    if (warp < NXP && lane == 0) {
                        const int off = warp < JT ? c.b[l] + warp : c.wf + warp - JT;
                        const float m1 = p.b1 * mb[l] + p.omb1 * ex;
                        const float m2 = p.b2 * vb[l] + p.omb2 * (ex * ex);
                        mb[l] = m1;
                        vb[l] = m2;
                        sm[pn + off] = sm[po + off] - adam_step(lrc * m1, m2 * ic2, p.eps);
                    }
                    // lane = 16 tile + 4 j + q: weight (j, column 4 ct + q) of tile ct
                    const int gi = lane & 15, ct = warp + NW * (lane >> 4);
                    const int off = (gi >> 2) * sw + 4 * ct + (gi & 3);
                    const float gsum = gv[0];
                    const float m1 = p.b1 * mw[l][0] + p.omb1 * gsum;
                    const float m2 = p.b2 * vw[l][0] + p.omb2 * (gsum * gsum);
                    mw[l][0] = m1;
                    vw[l][0] = m2;
                    sm[pn + c.w[l] + off] = sm[po + c.w[l] + off] - adam_step(lrc * m1, m2 * ic2, p.eps);
                }
#pragma unroll
                for (int tw = 0; tw < (PAIR ? 0 : TPW); ++tw) {
                    // warp -> column tile ct (4 columns) x neuron group jg
                    // (JPB neurons): JS = NW / NC groups cover all warps
                    constexpr int JS = NCL >= NW ? 1 : NW / NCL;
                    constexpr int JPB = JT / JS;
                    const int ct = NCL > NW ? warp + NW * tw : warp % NCL;
                    const int jg = NCL > NW ? 0 : warp / NCL, r = 4 * lane;
                    const int j0 = jg * JPB;
                    f2_t acc[JPB][4], sb[JPB], sf[JPB];
#pragma unroll
                    for (int j = 0; j < JPB; ++j) {
                        sb[j] = sf[j] = 0ull;
#pragma unroll
                        for (int q = 0; q < 4; ++q) acc[j][q] = 0ull;
                    }
                    ulonglong2 x[4];
                    if constexpr ((kPre || kPre1) && l == 1) {
#pragma unroll
                        for (int q = 0; q < 4; ++q) x[q] = bx[q];
                    } else {
#pragma unroll
                        for (int q = 0; q < 4; ++q) x[q] = *reinterpret_cast<const ulonglong2 *>(in + (4 * ct + q) * kSR + r);
                    }
                    float4 y4 = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (top) y4 = *reinterpret_cast<const float4 *>(dyp + r);
                    const f2_t one = f2_bcast(1.0f);
#pragma unroll
                    for (int j = 0; j < JPB; ++j) {
                        float4 z;
                        if constexpr (kPre && l == 1)
                            z = bz[j];
                        else
                            z = *reinterpret_cast<const float4 *>(zsrc + (j0 + j) * kSR + r);
                        if (top) {  // dZ_N = (a_N > 0) dy w_j on the fly (:102-107)
                            ffma2(sf[j], f2_pack(z.x, z.y), f2_pack(y4.x, y4.y));
                            ffma2(sf[j], f2_pack(z.z, z.w), f2_pack(y4.z, y4.w));
                            const float f = wfp[j0 + j];
                            z = make_float4(z.x > 0.f ? y4.x * f : 0.f, z.y > 0.f ? y4.y * f : 0.f,
                                            z.z > 0.f ? y4.z * f : 0.f, z.w > 0.f ? y4.w * f : 0.f);
                        }
                        const f2_t za = f2_pack(z.x, z.y), zb = f2_pack(z.z, z.w);
                        ffma2(sb[j], za, one);
                        ffma2(sb[j], zb, one);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            ffma2(acc[j][q], za, x[q].x);
                            ffma2(acc[j][q], zb, x[q].y);
                        }
                    }
                    float gv[4 * JPB];
#pragma unroll
                    for (int j = 0; j < JPB; ++j)
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const float2 h = f2_unpack(acc[j][q]);
                            gv[4 * j + q] = h.x + h.y;
                        }
                    // biases (and, top layer, final weights): with every warp
                    // holding all JT neurons (JS == 1) warp w reduces extra w
                    // inside its weight-gradient reduction, so no warp carries
                    // a second reduction chain; otherwise the column-tile-0 / -1
                    // warps reduce them afterwards
                    constexpr int NX = (l == NL ? 2 : 1) * JT;
                    constexpr bool XSPREAD = JS == 1 && TPW == 1 && NX <= NW;
                    if constexpr (XSPREAD) {
                        float ex = 0.f;  // register arrays: select, no dynamic index
#pragma unroll
                        for (int j = 0; j < JPB; ++j) {
                            if (warp == j) {
                                const float2 h = f2_unpack(sb[j]);
                                ex = h.x + h.y;
                            }
                            if (top && warp == JT + j) {
                                const float2 h = f2_unpack(sf[j]);
                                ex = h.x + h.y;
                            }
                        }
                        reduce_scatter_x<4 * JPB, 4 * JPB, 32>(gv, ex, lane);
                        if (warp < NX && lane == 0) {
                            const int off = warp < JT ? c.b[l] + warp : c.wf + warp - JT;
                            const float m1 = p.b1 * mb[l] + p.omb1 * ex;
                            const float m2 = p.b2 * vb[l] + p.omb2 * (ex * ex);
                            mb[l] = m1;
                            vb[l] = m2;
                            sm[pn + off] = sm[po + off] - adam_step(lrc * m1, m2 * ic2, p.eps);
                        }
                    } else {
                        reduce_scatter<4 * JPB, 4 * JPB, 32>(gv, lane);
                    }
                    constexpr int GSH = 5 - ilog2c(4 * JPB);  // replicas: 2^GSH lanes per weight
                    const int gi = lane >> GSH;                // j * 4 + q within the group
                    if ((lane & ((1 << GSH) - 1)) == 0) {
                        const int off = (j0 + (gi >> 2)) * sw + 4 * ct + (gi & 3);
                        const float gsum = gv[0];
                        const float m1 = p.b1 * mw[l][tw] + p.omb1 * gsum;
                        const float m2 = p.b2 * vw[l][tw] + p.omb2 * (gsum * gsum);
                        mw[l][tw] = m1;
                        vw[l][tw] = m2;
                        sm[pn + c.w[l] + off] = sm[po + c.w[l] + off] - adam_step(lrc * m1, m2 * ic2, p.eps);
                    }
                    // biases on the column-tile-0 warps, final weights (top layer)
                    // on the column-tile-1 warps: the extra reductions are spread
                    if (!XSPREAD && (ct == 0 || (top && ct == 1))) {
                        float bv[JPB];
#pragma unroll
                        for (int j = 0; j < JPB; ++j) {
                            const float2 h = f2_unpack(ct == 0 ? sb[j] : sf[j]);
                            bv[j] = h.x + h.y;
                        }
                        reduce_scatter<JPB, JPB, 32>(bv, lane);
                        constexpr int BSH = 5 - ilog2c(JPB);
                        const int bi = lane >> BSH;
                        if ((lane & ((1 << BSH) - 1)) == 0) {
                            const int off = (ct == 0 ? c.b[l] : c.wf) + j0 + bi;
                            const float gsum = bv[0];
                            const float m1 = p.b1 * mb[l] + p.omb1 * gsum;
                            const float m2 = p.b2 * vb[l] + p.omb2 * (gsum * gsum);
                            mb[l] = m1;
                            vb[l] = m2;
                            sm[pn + off] = sm[po + off] - adam_step(lrc * m1, m2 * ic2, p.eps);
                        }
                    }
                }
                if constexpr (LDA && l == 2) {
                    // dZ1 complete, the own W2 rows / final weights of step s+1 written
                    __syncthreads();
                    if (s >= 1 && tid == 0) mbar_arm(s2u(bars + c.wtbar + (s & 1)), wtbytes);  // step s+2
                    if (s + 1 < c.total && tid < CS * (JT + 1)) {
                        // to peer p: W2[own i][p's 4 columns] (k < JT), own final weights (k == JT)
                        const int pp = tid / (JT + 1), k = tid % (JT + 1), nb = (s + 1) & 1;
                        const float *src = k < JT ? sm + pn + c.w[2] + k * c.sw[2] + JT * pp : sm + pn + c.wf;
                        const uint32_t dst = k < JT ? s2u(sm + c.wt + (nb * H + rank * JT + k) * 4)
                                                    : s2u(sm + c.wfa + nb * H + rank * JT);
                        st_async4(mapa(dst, pp), *reinterpret_cast<const float4 *>(src), mapa(s2u(bars + c.wtbar + nb), pp));
                    }
                }
                if (l > 1 && !LDA) {
                    // receive: dZ_{l-1} own = (a_{l-1} > 0) * sum_q partial_q (:107)
                    const uint32_t rb = s2u(bars + 3 + 2 * (l - 2));
                    NOMA_TL(13)
                    if constexpr (kPre1 && l == 2) {  // layer 1's weight-gradient inputs, ahead of the wait
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            bx[q] = *reinterpret_cast<const ulonglong2 *>(XT + (4 * warp + q) * kSR + 4 * lane);
                    }
                    mbar_wait(rb, (uint32_t)(s & 1));
                    NOMA_TL(14)
                    if constexpr (JT * 64 == kLT) {  // all threads, two rows each (C2 -39 us vs 4 warps x 4 rows)
                        const int j = tid >> 6, r = 2 * (tid & 63);
                        const float *rs_ = sm + c.rsb[l - 1] + j * kSR + r;
                        float2 sum = *reinterpret_cast<const float2 *>(rs_);
#pragma unroll
                        for (int q = 1; q < CS; ++q) {
                            const float2 v = *reinterpret_cast<const float2 *>(rs_ + q * JT * kSR);
                            sum.x += v.x;
                            sum.y += v.y;
                        }
                        float2 *ap = reinterpret_cast<float2 *>(sm + c.aloc[l - 1] + j * kSR + r);
                        const float2 a = *ap;
                        *ap = make_float2(a.x > 0.f ? sum.x : 0.f, a.y > 0.f ? sum.y : 0.f);
                    } else if (tid < JT * 32) {
                        const int j = tid >> 5, r = 4 * lane;
                        const float *rs_ = sm + c.rsb[l - 1] + j * kSR + r;
                        float4 sum = *reinterpret_cast<const float4 *>(rs_);
#pragma unroll
                        for (int q = 1; q < CS; ++q) {
                            const float4 v = *reinterpret_cast<const float4 *>(rs_ + q * JT * kSR);
                            sum.x += v.x;
                            sum.y += v.y;
                            sum.z += v.z;
                            sum.w += v.w;
                        }
                        float4 *ap = reinterpret_cast<float4 *>(sm + c.aloc[l - 1] + j * kSR + r);
                        const float4 a = *ap;
                        *ap = make_float4(a.x > 0.f ? sum.x : 0.f, a.y > 0.f ? sum.y : 0.f,
                                          a.z > 0.f ? sum.z : 0.f, a.w > 0.f ? sum.w : 0.f);
                    }
                    __syncthreads();
                    if (tid == 0) mbar_arm(rb, rsbytes);
                }
            });
            NOMA_LPHASE(5)
            NOMA_TL(8)
            NOMA_GT(6)
            if (s + 1 < total) load_fx(s + 1);
            __syncthreads();
            NOMA_LPHASE(6)
            NOMA_TL(9)
        }
        // ---- epoch loss (hybrid_nn.cpp:190-192): trace[e] = sum r^2 / n -------
        if (c.ehist >= 0) {
            if (rank == 0 && p.trace && tid < kBatchRows) sm[c.ehist + e * kBatchRows + tid] = loss_acc;
        } else if (rank == 0 && p.trace) {
            if (tid < kBatchRows) sm[c.red + tid] = loss_acc;
            __syncthreads();
            if (tid == 0) {
                double t = 0.0;
                for (int i = 0; i < kBatchRows; ++i) t += sm[c.red + i];
                p.trace[(size_t)net * p.epochs + e] = t / (double)n;
            }
            __syncthreads();
        }
        loss_acc = 0.0f;
    }
    if (c.ehist >= 0 && rank == 0 && p.trace) {  // same order as the per-epoch sum
        __syncthreads();
        for (int e = tid; e < p.epochs; e += kLT) {
            double t = 0.0;
            for (int i = 0; i < kBatchRows; ++i) t += sm[c.ehist + e * kBatchRows + i];
            p.trace[(size_t)net * p.epochs + e] = t / (double)n;
        }
    }
    NOMA_LPHASE(7)
#ifdef NOMA_PROBES
    if (clk_on)
        for (int i = 0; i < 8; ++i) p.clocks[i] = clk_acc[i];
#else
    (void)clk_on;
    (void)clk_acc;
    (void)clk_prev;
    (void)tl;
#endif
#undef NOMA_LPHASE
    // ---- own slice of the trained parameters back to the FusedPlan layout ----
    const int pf = (total & 1) * c.npar;  // copy written by the last step
    float *pout = p.plans + (size_t)net * g.plan_total;
#pragma unroll
    for (int l = 1; l <= NL; ++l) {
        const int C = g.dims[l - 1];
        for (int i = tid; i < JT * C; i += kLT) {
            const int j = i / C, k = i - j * C;
            pout[g.plan_w[l] + (rank * JT + j) * g.plan_pad[l - 1] + k] = sm[pf + c.w[l] + j * c.sw[l] + k];
        }
        if (tid < JT) pout[g.plan_b[l] + rank * JT + tid] = sm[pf + c.b[l] + tid];
    }
    if (tid < JT) pout[g.plan_f + rank * JT + tid] = sm[pf + c.wf + tid];
    cl_sync();  // no CTA leaves while a peer could still address its shared memory
}

// Per-step minibatch tiles for the latency kernel: block (net, step) writes
// the feature-major tile X[width][kSR] of the rows perm[e][start..start+bsz)
// (zero rows past the batch), IQ-widened (iq_transform.cpp:17-20), and their
// r0 targets; the training kernel then moves a whole tile with one bulk copy.
// W = compile-time width (32, 64): the thread's row is read as W/4
// independent float4 loads and the odd rows' IQ rotation is applied from
// registers (W = 0: any width, one scalar load per element)
template <int W>
__global__ void __launch_bounds__(kBatchRows) lat_prep_kernel(TrainParams p, int total) {
    const int job = blockIdx.x, net = job / total, step = job - net * total;
    const int spe = (p.rows + p.batch - 1) / p.batch;
    const int e = step / spe, start = (step - e * spe) * p.batch, bsz = min(p.batch, p.rows - start);
    const int r = threadIdx.x, n = p.rows, width = p.width, M = width / 2, d = net / p.K;
    const bool wid = p.layout == NOMA_LAYOUT_WIDEN_COMPLEX;
    const int idx = r < bsz ? (int)p.perm[((size_t)net * p.epochs + e) * n + start + r] : -1;
    float *xo = p.xprep + (size_t)job * width * kSR;
    p.r0prep[(size_t)job * kBatchRows + r] = idx >= 0 ? p.r0[(size_t)net * n + idx] : 0.0f;
    const float *src = idx < 0 ? nullptr
                       : wid ? p.design32 + ((size_t)d * (n >> 1) + (idx >> 1)) * width
                             : p.design32 + ((size_t)d * n + idx) * width;
    const bool odd = wid && idx >= 0 && (idx & 1);
    if constexpr (W > 0) {
        float v[W];
#pragma unroll
        for (int q = 0; q < W / 4; ++q) {
            const float4 f = src ? reinterpret_cast<const float4 *>(src)[q] : make_float4(0.f, 0.f, 0.f, 0.f);
            v[4 * q] = f.x;
            v[4 * q + 1] = f.y;
            v[4 * q + 2] = f.z;
            v[4 * q + 3] = f.w;
        }
#pragma unroll
        for (int k = 0; k < W; ++k)  // widened odd row (iq_transform.cpp:17-20): [Im; -Re]
            xo[k * kSR + r] = !odd ? v[k] : (k < W / 2 ? v[W / 2 + k] : -v[k - W / 2]);
    } else {
        for (int k = 0; k < width; ++k) {
            float v = 0.0f;
            if (src) v = !odd ? src[k] : (k < M ? src[M + k] : -src[k - M]);
            xo[k * kSR + r] = v;
        }
    }
    if (r < kSR - kBatchRows)
        for (int k = 0; k < width; ++k) xo[k * kSR + kBatchRows + r] = 0.0f;
}

// host: pick the cluster size, carve shared memory, launch.  Returns
// NOMA_ERR_UNSUPPORTED when latency mode does not apply (caller falls back).
int train_lat_launch(TrainParams &p, cudaStream_t st) {
    if (p.batch < 1 || p.batch > kBatchRows || p.n_nets < 1) return NOMA_ERR_UNSUPPORTED;
    if (!p.xprep || !p.r0prep) return NOMA_ERR_UNSUPPORTED;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int want = 0;
    if (const char *f = std::getenv("NOMA_LAT_CLUSTER")) want = std::atoi(f);
    if (want == 1) return NOMA_ERR_UNSUPPORTED;
    const long total = (long)((p.rows + p.batch - 1) / p.batch) * p.epochs;
    if (total < 1 || total > kLatMaxSteps) return NOMA_ERR_UNSUPPORTED;
    if ((size_t)p.n_nets * total * p.width * kSR > p.prep_floats) return NOMA_ERR_UNSUPPORTED;
    bool prepped = false;  // the tiles are built once, for the first shape that fits
    const int cand[3] = {16, 8, 4};
    for (int ci = 0; ci < 3; ++ci) {
        const int cs = cand[ci];
        if (want && cs != want) continue;
        if (!want && p.n_nets * cs > sms) continue;
        LatCarve c;
        if (!lat_carve(p.g, cs, p.width, (int)total, p.epochs, &c)) continue;
        const size_t smem = (size_t)c.end * sizeof(float);
        if (!prepped) {
            const unsigned jobs = (unsigned)(p.n_nets * total);
            if (p.width == 32)
                lat_prep_kernel<32><<<jobs, kBatchRows, 0, st>>>(p, (int)total);
            else if (p.width == 64)
                lat_prep_kernel<64><<<jobs, kBatchRows, 0, st>>>(p, (int)total);
            else
                lat_prep_kernel<0><<<jobs, kBatchRows, 0, st>>>(p, (int)total);
            if (cudaGetLastError() != cudaSuccess) return NOMA_ERR_CUDA;
            prepped = true;
        }
        auto launch = [&](auto kern, int nwarps) -> int {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (cs > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(p.n_nets * cs);
            cfg.blockDim = dim3(nwarps * 32);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = cs;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            int nclusters = 0;
            if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) != cudaSuccess || nclusters < 1) {
                cudaGetLastError();
                return NOMA_ERR_UNSUPPORTED;
            }
            if (cudaLaunchKernelEx(&cfg, kern, p, c) != cudaSuccess) {
                cudaGetLastError();
                return NOMA_ERR_UNSUPPORTED;
            }
            return NOMA_OK;
        };
        const int vw = p.width <= 32 ? 2 : 4;  // float4 per gather thread
        // 8 warps for one hidden layer over a 32-wide input (less issue
        // contention on the critical path); NOMA_LAT_WARPS=16 overrides
        const bool nw8_ok = vw == 2;  // 32-wide input: k split and column tiles fit 8 warps
        int nw = nw8_ok ? 8 : 16;
        if (const char *f = std::getenv("NOMA_LAT_WARPS")) nw = std::atoi(f) == 8 && nw8_ok ? 8 : 16;
        auto pick = [&](auto cs_t, auto jt_t) -> int {
            constexpr int CS = decltype(cs_t)::value, JT = decltype(jt_t)::value;
            if (c.N == 1) {
                if (vw == 2) return nw == 8 ? launch(train_lat_kernel<CS, JT, 1, 2, 8>, 8)
                                            : launch(train_lat_kernel<CS, JT, 1, 2, 16>, 16);
                return launch(train_lat_kernel<CS, JT, 1, 4, 16>, 16);
            }
            if constexpr (JT >= 4 && CS * JT <= 64) {
                if (vw == 2) return nw == 8 ? launch(train_lat_kernel<CS, JT, 2, 2, 8>, 8)
                                            : launch(train_lat_kernel<CS, JT, 2, 2, 16>, 16);
                return launch(train_lat_kernel<CS, JT, 2, 4, 16>, 16);
            }
            return NOMA_ERR_UNSUPPORTED;
        };
        using I16 = std::integral_constant<int, 16>;
        using I8 = std::integral_constant<int, 8>;
        using I4 = std::integral_constant<int, 4>;
        using I2 = std::integral_constant<int, 2>;
        int r = NOMA_ERR_UNSUPPORTED;
        if (cs == 16 && c.jt == 2) r = pick(I16(), I2());
        else if (cs == 16 && c.jt == 4) r = pick(I16(), I4());
        else if (cs == 16 && c.jt == 8) r = pick(I16(), I8());
        else if (cs == 8 && c.jt == 4) r = pick(I8(), I4());
        else if (cs == 8 && c.jt == 8) r = pick(I8(), I8());
        else if (cs == 4 && c.jt == 8) r = pick(I4(), I8());
        if (r == NOMA_OK) {
            p.mode = 100 + cs;
            return NOMA_OK;
        }
    }
    return NOMA_ERR_UNSUPPORTED;
}

}  // namespace noma_dev
