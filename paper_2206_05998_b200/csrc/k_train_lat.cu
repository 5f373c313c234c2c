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
//     pass and the reduce-scatter of dA_l = W_{l+1}^T dZ_{l+1} in the backward.
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

#include "kernels.cuh"
#include "tiles.cuh"

namespace noma_dev {

namespace {

constexpr int kLT = 512;      // threads per CTA
constexpr int kLatMaxV = 4;   // float4 per gather thread: input width <= 64

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
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "NOMA_MBW_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
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

}  // namespace

// Shared-memory carve-up (floats), identical on host and device.
struct LatCarve {
    int cs, N, J[NOMA_MAX_DIMS], cin[NOMA_MAX_DIMS], sw[NOMA_MAX_DIMS], rsp[NOMA_MAX_DIMS];
    int xt, r0b, yall, dy, red, misc;
    int w[NOMA_MAX_DIMS], b[NOMA_MAX_DIMS], wf, npar;  // own parameters
    int m1, m2;                                        // Adam moments
    int aN;                                            // own a_N [J_N][kSR]
    int aloc[NOMA_MAX_DIMS], af[NOMA_MAX_DIMS], rsb[NOMA_MAX_DIMS];  // l < N
    int part[NOMA_MAX_DIMS], partb[NOMA_MAX_DIMS];     // weight-gradient partials
    int bars;                                          // mbarriers (8-byte aligned)
    int nbars, end;
};

__host__ __device__ inline int lat_pow2_floor(int v) {
    int p = 1;
    while (p * 2 <= v) p *= 2;
    return p;
}

// Returns false when the shape is outside this kernel (caller falls back).
__host__ __device__ inline bool lat_carve(const NetGeom &g, int cs, int width, LatCarve *c) {
    const int N = g.nd - 1;
    if (N < 1 || cs < 2 || cs > 16) return false;
    if (width != g.dims[0] || width % 8 || width > 4 * 4 * kLatMaxV) return false;
    c->cs = cs;
    c->N = N;
    for (int l = 1; l <= N; ++l) {
        if (g.dims[l] % cs) return false;
        c->J[l] = g.dims[l] / cs;
        c->cin[l] = g.dims[l - 1];
        if (c->J[l] % 2 || c->cin[l] % 4) return false;
        if (l < N && c->J[l] % 4) return false;
        c->sw[l] = c->cin[l] + 4;
        const int ntile = (c->J[l] / 2) * (c->cin[l] / 4);
        int r = ntile >= kLT ? 1 : lat_pow2_floor(kLT / ntile);
        c->rsp[l] = r > 32 ? 32 : r;
    }
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
    c->misc = off;
    off += 4;
    int np = 0;
    for (int l = 1; l <= N; ++l) {
        c->w[l] = off + np;
        np += c->J[l] * c->sw[l];
        c->b[l] = off + np;
        np += c->J[l];
    }
    c->wf = off + np;
    np += c->J[N];
    np = pad_to(np, 4);
    c->npar = np;
    off += np;
    c->m1 = off;
    off += np;
    c->m2 = off;
    off += np;
    c->aN = off;
    off += c->J[N] * kSR;
    for (int l = 1; l < N; ++l) {
        c->aloc[l] = off;
        off += c->J[l] * kSR;
        c->af[l] = off;
        off += g.dims[l] * kSR;
        c->rsb[l] = off;
        off += cs * c->J[l] * kSR;
    }
    for (int l = 1; l <= N; ++l) {
        c->part[l] = off;
        off += c->rsp[l] * c->J[l] * c->cin[l];
        c->partb[l] = off;
        off += c->rsp[l] * c->J[l] * 2;
    }
    off = pad_to(off, 2);
    c->bars = off;
    c->nbars = 2 + 2 * (N - 1);  // Y[2], AG_l, RS_l
    off += 2 * c->nbars;
    c->end = off;
    return (size_t)off * sizeof(float) <= 227 * 1024;
}

template <int CS>
__global__ void __launch_bounds__(kLT, 1) train_lat_kernel(TrainParams p, LatCarve c) {
    extern __shared__ __align__(16) float sm[];
    const int net = blockIdx.x / CS;
    if (p.status && p.status[net] != NOMA_OK) return;  // uniform over the cluster
    const uint32_t rank = cl_rank();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const NetGeom &g = p.g;
    const int N = c.N;
    const int n = p.rows, d = net / p.K, width = p.width, M = width / 2;
    const bool wid = p.layout == NOMA_LAYOUT_WIDEN_COMPLEX;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + c.bars);
    // barrier indices: Y[0], Y[1], then AG_l = 2 + 2(l-1), RS_l = 3 + 2(l-1)
    const bool clk_on = p.clocks && blockIdx.x == 0 && tid == 0;
    long long clk_acc[6] = {0, 0, 0, 0, 0, 0}, clk_prev = clk_on ? clock64() : 0;
#define NOMA_LPHASE(I)                               \
    if (clk_on) {                                    \
        const long long now = clock64();             \
        clk_acc[I] += now - clk_prev;                \
        clk_prev = now;                              \
    }

    for (int i = tid; i < c.bars; i += kLT) sm[i] = 0.0f;
    // own parameters from the FusedPlan buffer (fused_inference.cpp:19-42)
    const float *pl = p.plans + (size_t)net * g.plan_total;
    for (int l = 1; l <= N; ++l) {
        const int J = c.J[l], C = c.cin[l];
        for (int i = tid; i < J * C; i += kLT) {
            const int j = i / C, k = i % C;
            sm[c.w[l] + j * c.sw[l] + k] = pl[g.plan_w[l] + (rank * J + j) * g.plan_pad[l - 1] + k];
        }
        for (int j = tid; j < J; j += kLT) sm[c.b[l] + j] = pl[g.plan_b[l] + rank * J + j];
    }
    for (int j = tid; j < c.J[N]; j += kLT) sm[c.wf + j] = pl[g.plan_f + rank * c.J[N] + j];
    const uint32_t ybytes = CS * kBatchRows * 4;
    if (tid == 0) {
        for (int b = 0; b < c.nbars; ++b) mbar_init(s2u(bars + b), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_arm(s2u(bars + 0), ybytes);
        mbar_arm(s2u(bars + 1), ybytes);
        for (int l = 1; l < N; ++l) {
            mbar_arm(s2u(bars + 2 + 2 * (l - 1)), g.dims[l] * kBatchRows * 4);
            mbar_arm(s2u(bars + 3 + 2 * (l - 1)), CS * c.J[l] * kBatchRows * 4);
        }
    }

    // ---- step schedule and the two-stage gather prefetch --------------------
    const int spe = (n + p.batch - 1) / p.batch;  // steps per epoch
    const long total = (long)spe * p.epochs;
    const int gr = tid >> 2, gh = tid & 3;         // gather: 4 threads per row
    const int nv = width / 4;                       // float4 per row
    auto step_row = [&](long s, int r, int &bsz) -> int {  // perm index or -1
        const int e = (int)(s / spe), start = (int)(s % spe) * p.batch;
        bsz = min(p.batch, n - start);
        if (r >= bsz) return -1;
        return p.perm[((size_t)net * p.epochs + e) * n + start + r];
    };
    float4 rowv[kLatMaxV];
    float rowr0 = 0.0f;
    auto load_row = [&](int idx) {
#pragma unroll
        for (int v = 0; v < kLatMaxV; ++v) {
            const int f = gh + 4 * v;
            float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
            if (idx >= 0 && f < nv) {
                const int col = 4 * f;
                const float *src = wid ? p.design32 + ((size_t)d * (n >> 1) + (idx >> 1)) * width
                                       : p.design32 + ((size_t)d * n + idx) * width;
                if (!wid || !(idx & 1)) {
                    x = *reinterpret_cast<const float4 *>(src + col);
                } else if (col < M) {
                    x = *reinterpret_cast<const float4 *>(src + M + col);
                } else {
                    const float4 t = *reinterpret_cast<const float4 *>(src + col - M);
                    x = make_float4(-t.x, -t.y, -t.z, -t.w);
                }
            }
            rowv[v] = x;
        }
        rowr0 = (idx >= 0 && gh == 0) ? p.r0[(size_t)net * n + idx] : 0.0f;
    };
    auto store_row = [&](int buf) {
        float *xt = sm + c.xt + buf * width * kSR;
#pragma unroll
        for (int v = 0; v < kLatMaxV; ++v) {
            const int f = gh + 4 * v;
            if (f < nv) {
                xt[(4 * f + 0) * kSR + gr] = rowv[v].x;
                xt[(4 * f + 1) * kSR + gr] = rowv[v].y;
                xt[(4 * f + 2) * kSR + gr] = rowv[v].z;
                xt[(4 * f + 3) * kSR + gr] = rowv[v].w;
            }
        }
        if (gh == 0) sm[c.r0b + buf * kBatchRows + gr] = rowr0;
    };
    int bsz_dummy;
    load_row(total > 0 ? step_row(0, gr, bsz_dummy) : -1);
    store_row(0);
    int idx_next = total > 1 ? step_row(1, gr, bsz_dummy) : -1;
    load_row(idx_next);                              // rows of step 1
    idx_next = total > 2 ? step_row(2, gr, bsz_dummy) : -1;  // indices of step 2
    __syncthreads();
    cl_sync();  // every CTA's barriers initialised before any st.async lands

    float loss_acc = 0.0f;
    long s = 0;
    NOMA_LPHASE(5)
    for (int e = 0; e < p.epochs; ++e) {
        for (int st = 0; st < spe; ++st, ++s) {
            const int buf = (int)(s & 1);
            const int start = st * p.batch, bsz = min(p.batch, n - start);
            const float *XT = sm + c.xt + buf * width * kSR;
            // ---- forward (hybrid_nn.cpp:60-72), own neurons ------------------
            for (int l = 1; l <= N; ++l) {
                const int J = c.J[l], C = c.cin[l];
                const float *in = l == 1 ? XT : sm + c.af[l - 1];
                const float *W = sm + c.w[l], *bias = sm + c.b[l];
                float *out = l == N ? sm + c.aN : sm + c.aloc[l];
                const int items = J * 32;
                int ks = items >= kLT ? 1 : lat_pow2_floor(kLT / items);
                if (ks > C / 4) ks = lat_pow2_floor(C / 4);
                const int kchunks = C / 4;
                for (int t = tid; t < items * ks; t += kLT) {
                    const int kq = t % ks, rq = (t / ks) & 31, j = t / (ks * 32);
                    const int r0 = 4 * rq;
                    f2_t a0 = 0ull, a1 = 0ull;
                    const float *wr = W + j * c.sw[l];
                    for (int kc = kq; kc < kchunks; kc += ks) {
                        const float4 w4 = *reinterpret_cast<const float4 *>(wr + 4 * kc);
                        const float *ip = in + 4 * kc * kSR + r0;
                        const ulonglong2 x0 = *reinterpret_cast<const ulonglong2 *>(ip);
                        const ulonglong2 x1 = *reinterpret_cast<const ulonglong2 *>(ip + kSR);
                        const ulonglong2 x2 = *reinterpret_cast<const ulonglong2 *>(ip + 2 * kSR);
                        const ulonglong2 x3 = *reinterpret_cast<const ulonglong2 *>(ip + 3 * kSR);
                        f2_t wb = f2_bcast(w4.x);
                        ffma2(a0, wb, x0.x);
                        ffma2(a1, wb, x0.y);
                        wb = f2_bcast(w4.y);
                        ffma2(a0, wb, x1.x);
                        ffma2(a1, wb, x1.y);
                        wb = f2_bcast(w4.z);
                        ffma2(a0, wb, x2.x);
                        ffma2(a1, wb, x2.y);
                        wb = f2_bcast(w4.w);
                        ffma2(a0, wb, x3.x);
                        ffma2(a1, wb, x3.y);
                    }
                    float2 u = f2_unpack(a0), v = f2_unpack(a1);
                    for (int o = 1; o < ks; o <<= 1) {  // butterfly over the k split
                        u.x += __shfl_xor_sync(0xffffffffu, u.x, o);
                        u.y += __shfl_xor_sync(0xffffffffu, u.y, o);
                        v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
                        v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
                    }
                    const float bj = bias[j];
                    const float4 y = make_float4(fmaxf(u.x + bj, 0.f), fmaxf(u.y + bj, 0.f),
                                                 fmaxf(v.x + bj, 0.f), fmaxf(v.y + bj, 0.f));
                    if (kq == 0) *reinterpret_cast<float4 *>(out + j * kSR + r0) = y;
                    if (l < N) {  // all-gather: lane kq sends to ranks kq, kq+ks, ...
                        const uint32_t la = s2u(sm + c.af[l] + (rank * J + j) * kSR + r0);
                        const uint32_t lb = s2u(bars + 2 + 2 * (l - 1));
                        for (int q = kq; q < CS; q += ks) st_async4(mapa(la, q), y, mapa(lb, q));
                    }
                }
                if (l < N) {
                    const uint32_t lb = s2u(bars + 2 + 2 * (l - 1));
                    mbar_wait(lb, (uint32_t)(s & 1));
                    // re-arm for step s+1 (its bytes cannot land before every
                    // CTA has finished step s)
                    if (tid == 0) mbar_arm(lb, g.dims[l] * kBatchRows * 4);
                }
            }
            __syncthreads();
            NOMA_LPHASE(0)
            // ---- final-layer partials to every CTA; gather the next tile ------
            const uint32_t ybar = s2u(bars + buf);
            if (warp == 0) {
                const int r0 = 4 * lane;
                const float *aN = sm + c.aN;
                const float *wf = sm + c.wf;
                float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
                for (int j = 0; j < c.J[N]; ++j) {
                    const float4 a = *reinterpret_cast<const float4 *>(aN + j * kSR + r0);
                    const float f = wf[j];
                    y.x = fmaf(f, a.x, y.x);
                    y.y = fmaf(f, a.y, y.y);
                    y.z = fmaf(f, a.z, y.z);
                    y.w = fmaf(f, a.w, y.w);
                }
                const uint32_t la = s2u(sm + c.yall + (buf * CS + rank) * kBatchRows + r0);
#pragma unroll
                for (int q = 0; q < CS; ++q) st_async4(mapa(la, q), y, mapa(ybar, q));
            }
            if (s + 1 < total) {
                store_row(buf ^ 1);  // rows of step s+1 (loaded one step ago)
                load_row(idx_next);  // rows of step s+2
                idx_next = s + 3 < total ? step_row(s + 3, gr, bsz_dummy) : -1;
            }
            if (tid == kLT - 1) {  // Adam bias corrections (FP64 pow, hybrid_nn.cpp:133-135)
                const double c1 = 1.0 - pow(p.b1d, (double)(s + 1));
                const double c2 = 1.0 - pow(p.b2d, (double)(s + 1));
                sm[c.misc + 0] = (float)(p.lr_d / c1);
                sm[c.misc + 1] = (float)(1.0 / c2);
            }
            NOMA_LPHASE(1)
            // ---- residual a_N w - r0, dy = 2 r / B (hybrid_nn.cpp:94-98) --------
            if (tid < kBatchRows) {
                mbar_wait(ybar, (uint32_t)((s >> 1) & 1));
                const float *ya = sm + c.yall + buf * CS * kBatchRows + tid;
                float yh = 0.0f;
#pragma unroll
                for (int q = 0; q < CS; ++q) yh += ya[q * kBatchRows];
                const float res = tid < bsz ? yh - sm[c.r0b + buf * kBatchRows + tid] : 0.0f;
                sm[c.dy + tid] = (2.0f / (float)bsz) * res;
                loss_acc = fmaf(res, res, loss_acc);
            }
            __syncthreads();
            if (tid == 0) mbar_arm(ybar, ybytes);  // phase for step s+2
            NOMA_LPHASE(2)
            // ---- backward (hybrid_nn.cpp:99-112), own neurons ---------------
            for (int l = N; l >= 1; --l) {
                const int J = c.J[l], C = c.cin[l];
                const bool top = l == N;
                const float *zsrc = top ? sm + c.aN : sm + c.aloc[l];  // a_N, or dZ_l in place
                const float *dyp = sm + c.dy, *wf = sm + c.wf;
                const float *in = l == 1 ? XT : sm + c.af[l - 1];
                const int rsp = c.rsp[l], nct = C / 4;
                const int ntile = (J / 2) * nct;
                float *part = sm + c.part[l], *partb = sm + c.partb[l];
                for (int t = tid; t < ntile * rsp; t += kLT) {
                    const int rs = t % rsp, tile = t / rsp;
                    const int it = tile / nct, ct = tile % nct;
                    const int i0 = 2 * it, c0 = 4 * ct;
                    f2_t acc[2][4], sb[2], sf[2];
#pragma unroll
                    for (int a = 0; a < 2; ++a) {
                        sb[a] = sf[a] = 0ull;
#pragma unroll
                        for (int q = 0; q < 4; ++q) acc[a][q] = 0ull;
                    }
                    const float wf0 = top ? wf[i0] : 0.f, wf1 = top ? wf[i0 + 1] : 0.f;
                    const f2_t one = f2_bcast(1.0f);
                    for (int rq = rs; rq < 32; rq += rsp) {
                        const int r = 4 * rq;
                        float4 z0 = *reinterpret_cast<const float4 *>(zsrc + i0 * kSR + r);
                        float4 z1 = *reinterpret_cast<const float4 *>(zsrc + (i0 + 1) * kSR + r);
                        if (top) {  // dZ_N = (a_N > 0) dy w_j, formed on the fly (:102-107)
                            const float4 y = *reinterpret_cast<const float4 *>(dyp + r);
                            if (ct == 0) {  // final-layer gradient a_N^T dy (:99)
                                ffma2(sf[0], f2_pack(z0.x, z0.y), f2_pack(y.x, y.y));
                                ffma2(sf[0], f2_pack(z0.z, z0.w), f2_pack(y.z, y.w));
                                ffma2(sf[1], f2_pack(z1.x, z1.y), f2_pack(y.x, y.y));
                                ffma2(sf[1], f2_pack(z1.z, z1.w), f2_pack(y.z, y.w));
                            }
                            z0 = make_float4(z0.x > 0.f ? y.x * wf0 : 0.f, z0.y > 0.f ? y.y * wf0 : 0.f,
                                             z0.z > 0.f ? y.z * wf0 : 0.f, z0.w > 0.f ? y.w * wf0 : 0.f);
                            z1 = make_float4(z1.x > 0.f ? y.x * wf1 : 0.f, z1.y > 0.f ? y.y * wf1 : 0.f,
                                             z1.z > 0.f ? y.z * wf1 : 0.f, z1.w > 0.f ? y.w * wf1 : 0.f);
                        }
                        const f2_t z0a = f2_pack(z0.x, z0.y), z0b = f2_pack(z0.z, z0.w);
                        const f2_t z1a = f2_pack(z1.x, z1.y), z1b = f2_pack(z1.z, z1.w);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const ulonglong2 x = *reinterpret_cast<const ulonglong2 *>(in + (c0 + q) * kSR + r);
                            ffma2(acc[0][q], z0a, x.x);
                            ffma2(acc[0][q], z0b, x.y);
                            ffma2(acc[1][q], z1a, x.x);
                            ffma2(acc[1][q], z1b, x.y);
                        }
                        if (ct == 0) {  // bias gradient colsum dZ (:110)
                            ffma2(sb[0], z0a, one);
                            ffma2(sb[0], z0b, one);
                            ffma2(sb[1], z1a, one);
                            ffma2(sb[1], z1b, one);
                        }
                    }
#pragma unroll
                    for (int a = 0; a < 2; ++a) {
                        float v[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const float2 h = f2_unpack(acc[a][q]);
                            v[q] = h.x + h.y;
                        }
                        *reinterpret_cast<float4 *>(part + (rs * J + i0 + a) * C + c0) =
                            make_float4(v[0], v[1], v[2], v[3]);
                        if (ct == 0) {
                            const float2 hb = f2_unpack(sb[a]), hf = f2_unpack(sf[a]);
                            partb[(rs * J + i0 + a) * 2 + 0] = hb.x + hb.y;
                            partb[(rs * J + i0 + a) * 2 + 1] = hf.x + hf.y;
                        }
                    }
                }
                if (l > 1) {
                    // dA_{l-1} partial = sum_{j own} W_l[j][c] dZ_l[j][r] (:111) for
                    // every c, reduce-scattered to the owner of c.
                    const int Jd = c.J[l - 1];
                    const float *W = sm + c.w[l];
                    const uint32_t rb = s2u(bars + 3 + 2 * (l - 2));
                    for (int t = tid; t < (C / 4) * 32; t += kLT) {
                        const int rq = t & 31, cq = t >> 5;
                        const int r = 4 * rq, cc = 4 * cq;
                        f2_t acc[4][2];
#pragma unroll
                        for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = 0ull;
                        for (int j = 0; j < J; ++j) {
                            const float4 w4 = *reinterpret_cast<const float4 *>(W + j * c.sw[l] + cc);
                            float4 z = *reinterpret_cast<const float4 *>(zsrc + j * kSR + r);
                            if (top) {
                                const float4 y = *reinterpret_cast<const float4 *>(dyp + r);
                                const float f = wf[j];
                                z = make_float4(z.x > 0.f ? y.x * f : 0.f, z.y > 0.f ? y.y * f : 0.f,
                                                z.z > 0.f ? y.z * f : 0.f, z.w > 0.f ? y.w * f : 0.f);
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
                        const int owner = cc / Jd, lc = cc - owner * Jd;
                        const uint32_t la = s2u(sm + c.rsb[l - 1] + (rank * Jd + lc) * kSR + r);
                        const uint32_t ra = mapa(la, owner), rbar = mapa(rb, owner);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const float2 u = f2_unpack(acc[q][0]), v = f2_unpack(acc[q][1]);
                            st_async4(ra + q * kSR * 4, make_float4(u.x, u.y, v.x, v.y), rbar);
                        }
                    }
                    // receive: dZ_{l-1} own = (a_{l-1} > 0) * sum_q partial_q (:107)
                    mbar_wait(rb, (uint32_t)(s & 1));
                    const float *rs_ = sm + c.rsb[l - 1];
                    float *al = sm + c.aloc[l - 1];
                    for (int t = tid; t < Jd * 32; t += kLT) {
                        const int j = t >> 5, r = 4 * (t & 31);
                        float4 sum = *reinterpret_cast<const float4 *>(rs_ + j * kSR + r);
                        for (int q = 1; q < CS; ++q) {
                            const float4 v = *reinterpret_cast<const float4 *>(rs_ + (q * Jd + j) * kSR + r);
                            sum.x += v.x;
                            sum.y += v.y;
                            sum.z += v.z;
                            sum.w += v.w;
                        }
                        float4 *ap = reinterpret_cast<float4 *>(al + j * kSR + r);
                        const float4 a = *ap;
                        *ap = make_float4(a.x > 0.f ? sum.x : 0.f, a.y > 0.f ? sum.y : 0.f,
                                          a.z > 0.f ? sum.z : 0.f, a.w > 0.f ? sum.w : 0.f);
                    }
                    __syncthreads();
                    if (tid == 0) mbar_arm(rb, CS * Jd * kBatchRows * 4);
                }
            }
            __syncthreads();
            NOMA_LPHASE(3)
            // ---- Adam (hybrid_nn.cpp:118-144) over the own parameters ---------
            {
                const float lrc = sm[c.misc + 0], ic2 = sm[c.misc + 1];
                float *M1 = sm + c.m1, *M2 = sm + c.m2;
                int base = 0;
                for (int l = 1; l <= N + 1; ++l) {
                    const bool fin = l == N + 1;
                    const int L = fin ? N : l;
                    const int J = c.J[L], C = c.cin[L], rsp = c.rsp[L];
                    const int cnt = fin ? J : J * C + J;
                    const float *part = sm + c.part[L], *partb = sm + c.partb[L];
                    for (int i = tid; i < cnt; i += kLT) {
                        float gsum = 0.0f;
                        float *th;
                        if (fin) {
                            for (int q = 0; q < rsp; ++q) gsum += partb[(q * J + i) * 2 + 1];
                            th = sm + c.wf + i;
                        } else if (i < J * C) {
                            const int j = i / C, k = i % C;
                            for (int q = 0; q < rsp; ++q) gsum += part[(q * J + j) * C + k];
                            th = sm + c.w[L] + j * c.sw[L] + k;
                        } else {
                            const int j = i - J * C;
                            for (int q = 0; q < rsp; ++q) gsum += partb[(q * J + j) * 2 + 0];
                            th = sm + c.b[L] + j;
                        }
                        const int pi = base + i;
                        const float m1 = p.b1 * M1[pi] + p.omb1 * gsum;
                        const float m2 = p.b2 * M2[pi] + p.omb2 * (gsum * gsum);
                        M1[pi] = m1;
                        M2[pi] = m2;
                        *th -= __fdividef(lrc * m1, sqrtf(m2 * ic2) + p.eps);
                    }
                    base += cnt;
                }
            }
            __syncthreads();
            NOMA_LPHASE(4)
        }
        // ---- epoch loss (hybrid_nn.cpp:190-192): trace[e] = sum r^2 / n -------
        if (rank == 0 && p.trace) {
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
    NOMA_LPHASE(5)
    if (clk_on)
        for (int i = 0; i < 6; ++i) p.clocks[i] = clk_acc[i];
#undef NOMA_LPHASE
    // ---- own slice of the trained parameters back to the FusedPlan layout ----
    float *po = p.plans + (size_t)net * g.plan_total;
    for (int l = 1; l <= N; ++l) {
        const int J = c.J[l], C = c.cin[l];
        for (int i = tid; i < J * C; i += kLT) {
            const int j = i / C, k = i % C;
            po[g.plan_w[l] + (rank * J + j) * g.plan_pad[l - 1] + k] = sm[c.w[l] + j * c.sw[l] + k];
        }
        for (int j = tid; j < J; j += kLT) po[g.plan_b[l] + rank * J + j] = sm[c.b[l] + j];
    }
    for (int j = tid; j < c.J[N]; j += kLT) po[g.plan_f + rank * c.J[N] + j] = sm[c.wf + j];
    cl_sync();  // no CTA leaves while a peer could still address its shared memory
}

// host: pick the cluster size, carve shared memory, launch.  Returns
// NOMA_ERR_UNSUPPORTED when latency mode does not apply (caller falls back).
int train_lat_launch(TrainParams &p, cudaStream_t st) {
    if (p.batch < 1 || p.batch > kBatchRows || p.n_nets < 1) return NOMA_ERR_UNSUPPORTED;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int want = 0;
    if (const char *f = std::getenv("NOMA_LAT_CLUSTER")) want = std::atoi(f);
    if (want == 1) return NOMA_ERR_UNSUPPORTED;
    const int cand[4] = {16, 8, 4, 2};
    for (int ci = 0; ci < 4; ++ci) {
        const int cs = cand[ci];
        if (want && cs != want) continue;
        if (!want && p.n_nets * cs > sms) continue;
        LatCarve c;
        if (!lat_carve(p.g, cs, p.width, &c)) continue;
        const size_t smem = (size_t)c.end * sizeof(float);
        auto launch = [&](auto kern) -> int {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (cs > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(p.n_nets * cs);
            cfg.blockDim = dim3(kLT);
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
        int r = NOMA_ERR_UNSUPPORTED;
        switch (cs) {
            case 16: r = launch(train_lat_kernel<16>); break;
            case 8: r = launch(train_lat_kernel<8>); break;
            case 4: r = launch(train_lat_kernel<4>); break;
            default: r = launch(train_lat_kernel<2>); break;
        }
        if (r == NOMA_OK) {
            p.mode = 100 + cs;
            return NOMA_OK;
        }
    }
    return NOMA_ERR_UNSUPPORTED;
}

}  // namespace noma_dev
