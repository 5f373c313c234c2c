// FP64 pilot-phase training (the bit-consistent mode) for one hidden layer of
// 64 on a 32- or 64-wide input (C1, C5): hybrid_nn::train (hybrid_nn.cpp:
// 158-195) with loss_and_grad (:84-114) and adam_step (:118-144) in the
// reference's FP64 arithmetic, one 8-warp CTA per user network, register
// tiles of DFMA.
//
// k_train_f64.cu (the shape-general FP64 kernel) walks every product through
// shared memory and reaches ~2 % of the FP64 rate (0.9 of 37 TF/s).  Here:
//   * forward: 8 neurons x 4 rows of accumulators per thread, operands two
//     columns at a time (LDS.128 = two doubles), the linear branch x.w0 formed
//     alongside; the residual x w0 + a_N w - y as hybrid_nn.cpp:94 (no FP32
//     r0 shortcut);
//   * weight gradient gW = dZ^T X: 4 neurons x IN/16 columns per thread over
//     all 128 rows (no cross-thread reduction); the thread owns those
//     parameters and their FP64 Adam moments in registers for the whole
//     training; biases / final weights on threads 0-127 from fixed-order warp
//     partials;
//   * the next minibatch's pre-widened FP64 rows arrive by one bulk copy
//     each (mbarrier) while Adam runs.
// Summation orders are fixed (bit-reproducible runs); they differ from
// Eigen's, which FP64 absorbs (reordered-sum FP64 training stays within
// 1e-14 of the reference, profiles/r02_precision_probe.txt).
#include <cstdlib>

#include "kernels.cuh"

namespace noma_dev {

namespace {

constexpr int kW8dThreads = 256;
constexpr unsigned kFullD = 0xffffffffu;

template <int IN>
struct W8dGeom {
    static constexpr int XS = IN + 2;              // X row stride (doubles); rows 16-byte aligned
    static constexpr int WS = IN + 2;              // W row stride
    static constexpr int DS = kBatchRows + 2;      // DZ row stride
    static constexpr int off_x = 0;
    static constexpr int off_y = off_x + kBatchRows * XS;
    static constexpr int off_w = off_y + kBatchRows;
    static constexpr int off_b = off_w + 64 * WS;
    static constexpr int off_f = off_b + 64;
    static constexpr int off_w0 = off_f + 64;
    static constexpr int off_dz = off_w0 + IN;
    static constexpr int off_red = off_dz + 64 * DS;  // [8 warps][gf | gb][64]
    static constexpr int off_ls = off_red + 8 * 2 * 64;
    static constexpr int off_gbar = off_ls + kW8dThreads;  // mbarrier (minibatch rows), one double
    static constexpr int off_end = off_gbar + 1;
    static constexpr size_t bytes = (size_t)off_end * sizeof(double);
};

__device__ __forceinline__ void cp8d(double *dst, const double *src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_wait_d() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}
// minibatch rows by one bulk copy each (TMA engine) counted on an mbarrier
__device__ __forceinline__ uint32_t w8d_s2u(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void w8d_row_copy(double *dst, const double *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     w8d_s2u(dst)),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void w8d_bar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W8D_MBW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W8D_MBW_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ double shfl_xor_d(double v, int o) { return __shfl_xor_sync(kFullD, v, o); }
__device__ __forceinline__ double shfl_d(double v, int src) { return __shfl_sync(kFullD, v, src); }

}  // namespace

// Thread roles (warp w, q = lane >> 3, l8 = lane & 7):
//  forward   neurons j = l8 + 8m (m < 8), rows r_i = 16 w + q + 4i (i < 4);
//  residual  the reduce over the quarter's 8 lanes leaves row r_(l8 >> 1) on
//            lanes l8 and l8 ^ 1 (the even lane owns it);
//  gradient  neurons 8 w + 4 (q & 1) + n (n < 4), columns
//            (q >> 1) IN/2 + 16 t + 2 l8 + e (t < IN/32, e < 2), all 128 rows.
template <int IN>
__global__ void __launch_bounds__(kW8dThreads, 1)
    train_w8d_kernel(TrainF64Params p, const double *__restrict__ wide, const double *__restrict__ ctab) {
    using G = W8dGeom<IN>;
    constexpr int NT = IN / 32;  // column pairs per gradient thread (16 apart)
    extern __shared__ __align__(16) double smd[];
    const int net = blockIdx.x;
    if (p.status && p.status[net] != NOMA_OK) return;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, q = lane >> 3, l8 = lane & 7;
    const int n = p.rows, d = net / p.K, k_user = net - d * p.K;
    double *X = smd + G::off_x;
    double *Y = smd + G::off_y;
    double *W = smd + G::off_w;
    double *B = smd + G::off_b;
    double *F = smd + G::off_f;
    double *W0 = smd + G::off_w0;
    double *DZ = smd + G::off_dz;
    double *RED = smd + G::off_red;
    double *LS = smd + G::off_ls;

    // ---- parameters in: theta in the reference flat order (W_1 row-major, b_1,
    // final; hybrid_nn.hpp:15-23), w0 frozen ---------------------------------
    double *theta = p.theta + (size_t)net * p.ptrain;
    for (int i = tid; i < 64 * IN; i += kW8dThreads) W[(i / IN) * G::WS + i % IN] = theta[i];
    if (tid < 64) {
        B[tid] = theta[64 * IN + tid];
        F[tid] = theta[64 * IN + 64 + tid];
    }
    for (int c = tid; c < IN; c += kW8dThreads) W0[c] = p.w0[(size_t)net * IN + c];

    // gradient-thread ownership and FP64 Adam moments (fresh per train() call)
    const int gj0 = 8 * warp + 4 * (q & 1), gc0 = (q >> 1) * (IN / 2) + 2 * l8;
    double mw[4][NT][2], vw[4][NT][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int t = 0; t < NT; ++t) mw[a][t][0] = mw[a][t][1] = vw[a][t][0] = vw[a][t][1] = 0.0;
    double mb = 0.0, vb = 0.0;

    // minibatch copy: two threads per widened row (IN/2 doubles each) and the
    // row's target (hybrid_nn.cpp:180-187); zeros past the batch end
    const uint16_t *permn = p.perm + (size_t)net * p.epochs * n;
    const double *wrow = wide + (size_t)d * n * IN;
    const int grow = tid;  // thread r < 128: row r (one bulk copy) and its target
    auto target = [&](int row) -> const double * {
        return p.layout == NOMA_LAYOUT_WIDEN_COMPLEX
                   ? p.targets + (((size_t)d * (n / 2) + (row >> 1)) * p.K + k_user) * 2 + (row & 1)
                   : p.targets + ((size_t)d * p.K + k_user) * n + row;
    };
    // rows past the batch end keep the previous, finite values (their dZ is
    // zero) and start as zeros
    const uint32_t gbar = w8d_s2u(smd + G::off_gbar);
    for (int i = tid; i < kBatchRows * G::XS; i += kW8dThreads) X[i] = 0.0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // before the bulk copies overwrite
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(gbar) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto gather = [&](int idx, int nrows) {  // every thread; nrows valid rows
        if (tid == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(gbar),
                         "r"((uint32_t)nrows * IN * 8)
                         : "memory");
        if (grow < nrows) w8d_row_copy(X + grow * G::XS, wrow + (size_t)idx * IN, IN * 8, gbar);
        if (grow < kBatchRows) cp8d(Y + grow, target(grow < nrows ? idx : 0), grow < nrows);
    };
    uint32_t gphase = 0;
    {
        const int b0 = p.epochs > 0 ? min(p.batch, n) : 0;
        if (b0 > 0) {
            gather(grow < b0 ? permn[grow] : 0, b0);
            w8d_bar_wait(gbar, gphase);
            gphase ^= 1;
        }
        cp_wait_d();
    }
    __syncthreads();

    double lossacc = 0.0;
    int step = 0;
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
            const double c1 = ctab[2 * step], c2 = ctab[2 * step + 1];  // 1 - beta^t (host pow)

            // ---- forward: a = relu(W x + b) (hybrid_nn.cpp:60-67), x.w0 -----
            double acc[8][4], lin[4];
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const double bj = B[l8 + 8 * m];
#pragma unroll
                for (int i = 0; i < 4; ++i) acc[m][i] = bj;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) lin[i] = 0.0;
            {
                const double *xb = X + (16 * warp + q) * G::XS;
                const double *wb = W + l8 * G::WS;
#pragma unroll 1
                for (int k = 0; k < IN; k += 2) {
                    double2 w[8], x[4];
#pragma unroll
                    for (int m = 0; m < 8; ++m) w[m] = *reinterpret_cast<const double2 *>(wb + 8 * m * G::WS + k);
#pragma unroll
                    for (int i = 0; i < 4; ++i) x[i] = *reinterpret_cast<const double2 *>(xb + 4 * i * G::XS + k);
                    const double2 w0 = *reinterpret_cast<const double2 *>(W0 + k);
#pragma unroll
                    for (int m = 0; m < 8; ++m)
#pragma unroll
                        for (int i = 0; i < 4; ++i) acc[m][i] = fma(w[m].x, x[i].x, acc[m][i]);
#pragma unroll
                    for (int i = 0; i < 4; ++i) lin[i] = fma(x[i].x, w0.x, lin[i]);
#pragma unroll
                    for (int m = 0; m < 8; ++m)
#pragma unroll
                        for (int i = 0; i < 4; ++i) acc[m][i] = fma(w[m].y, x[i].y, acc[m][i]);
#pragma unroll
                    for (int i = 0; i < 4; ++i) lin[i] = fma(x[i].y, w0.y, lin[i]);
                }
            }
            // ReLU and the final dot a . w_final (hybrid_nn.cpp:81), partial
            // over this thread's 8 neurons for its 4 rows
            double yp[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const double fw = F[l8 + 8 * m];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    acc[m][i] = acc[m][i] > 0.0 ? acc[m][i] : 0.0;
                    yp[i] = fma(fw, acc[m][i], yp[i]);
                }
            }
            // reduce over the quarter's 8 lanes: rows split by lane bits 2, 1;
            // the last round sums the pair (l8, l8 ^ 1) -- row r_(l8 >> 1)
            double yh;
            {
                const bool b4 = l8 & 4, b2 = l8 & 2;
                double y2[2];
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    const double send = b4 ? yp[t] : yp[t + 2];
                    const double keep = b4 ? yp[t + 2] : yp[t];
                    y2[t] = keep + shfl_xor_d(send, 4);
                }
                const double send = b2 ? y2[0] : y2[1];
                const double keep = b2 ? y2[1] : y2[0];
                yh = keep + shfl_xor_d(send, 2);
                const double o = shfl_xor_d(yh, 1);  // lower + upper on both lanes
                yh = (l8 & 1) ? o + yh : yh + o;
            }
            // row of this lane pair: i = (l8 >> 2) * 2 + ((l8 >> 1) & 1) -> r_i
            const int ri = 2 * ((l8 >> 2) & 1) + ((l8 >> 1) & 1);
            double lin_r = lin[0];
#pragma unroll
            for (int i = 1; i < 4; ++i) lin_r = ri == i ? lin[i] : lin_r;
            const int row = 16 * warp + q + 4 * ri;
            // residual x w0 + a_N w - y (hybrid_nn.cpp:94); dy = (2 / B) r (:98)
            const bool valid = row < bsz;
            const double res = valid ? (lin_r + yh) - Y[row] : 0.0;
            const double dy_r = (2.0 / (double)bsz) * res;
            if (!(l8 & 1)) lossacc = fma(res, res, lossacc);
            double dy[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)  // row r_i lives on lanes (i>>1)*4 + (i&1)*2 (+1)
                dy[i] = shfl_d(dy_r, (lane & 24) | ((i >> 1) << 2) | ((i & 1) << 1));
            // dZ = (a > 0) ? dy w_f : 0 (:102, :107); g_final, g_b partials
            double gf[8], gb[8];
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int j = l8 + 8 * m;
                const double fw = F[j];
                gf[m] = gb[m] = 0.0;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const double z = acc[m][i] > 0.0 ? dy[i] * fw : 0.0;
                    gf[m] = fma(acc[m][i], dy[i], gf[m]);
                    gb[m] += z;
                    DZ[j * G::DS + 16 * warp + q + 4 * i] = z;
                }
            }
#pragma unroll
            for (int m = 0; m < 8; ++m) {  // over the 4 quarters, fixed order
                gf[m] += shfl_xor_d(gf[m], 8);
                gb[m] += shfl_xor_d(gb[m], 8);
                gf[m] += shfl_xor_d(gf[m], 16);
                gb[m] += shfl_xor_d(gb[m], 16);
            }
            if (q == 0) {
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    RED[warp * 128 + l8 + 8 * m] = gf[m];
                    RED[warp * 128 + 64 + l8 + 8 * m] = gb[m];
                }
            }
            __syncthreads();

            // ---- weight gradient gW = dZ^T X (hybrid_nn.cpp:109) --------------
            double ga[4][NT][2];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int t = 0; t < NT; ++t) ga[a][t][0] = ga[a][t][1] = 0.0;
            {
                const double *zb = DZ + gj0 * G::DS;
                const double *xb = X + gc0;
#pragma unroll 1
                for (int r = 0; r < kBatchRows; r += 2) {
                    double2 z[4];
#pragma unroll
                    for (int a = 0; a < 4; ++a) z[a] = *reinterpret_cast<const double2 *>(zb + a * G::DS + r);
#pragma unroll
                    for (int rr = 0; rr < 2; ++rr) {
                        double2 xv[NT];
#pragma unroll
                        for (int t = 0; t < NT; ++t)
                            xv[t] = *reinterpret_cast<const double2 *>(xb + (r + rr) * G::XS + 16 * t);
#pragma unroll
                        for (int a = 0; a < 4; ++a) {
                            const double za = rr ? z[a].y : z[a].x;
#pragma unroll
                            for (int t = 0; t < NT; ++t) {
                                ga[a][t][0] = fma(za, xv[t].x, ga[a][t][0]);
                                ga[a][t][1] = fma(za, xv[t].y, ga[a][t][1]);
                            }
                        }
                    }
                }
            }
            __syncthreads();  // X and DZ are dead

            // ---- next minibatch in flight while Adam runs ---------------------
            if (nb > 0) gather(nidx, nb);

            // ---- Adam (hybrid_nn.cpp:118-124): theta -= lr (m / c1) / (sqrt(v / c2) + eps)
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int t = 0; t < NT; ++t)
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const double gr = ga[a][t][u];
                        const double m1 = p.b1 * mw[a][t][u] + (1.0 - p.b1) * gr;
                        const double m2 = p.b2 * vw[a][t][u] + (1.0 - p.b2) * (gr * gr);
                        mw[a][t][u] = m1;
                        vw[a][t][u] = m2;
                        double &th = W[(gj0 + a) * G::WS + gc0 + 16 * t + u];
                        th -= p.lr * (m1 / c1) / (sqrt(m2 / c2) + p.eps);
                    }
            if (tid < 128) {  // biases (tid < 64), final weights: warps summed in order
                const int j = tid & 63, part = tid < 64 ? 64 : 0;
                double gsum = RED[part + j];
#pragma unroll
                for (int w = 1; w < 8; ++w) gsum += RED[w * 128 + part + j];
                double &th = tid < 64 ? B[j] : F[j];
                mb = p.b1 * mb + (1.0 - p.b1) * gsum;
                vb = p.b2 * vb + (1.0 - p.b2) * (gsum * gsum);
                th -= p.lr * (mb / c1) / (sqrt(vb / c2) + p.eps);
            }
            cp_wait_d();
            if (nb > 0) {
                w8d_bar_wait(gbar, gphase);
                gphase ^= 1;
            }
            ++step;
            __syncthreads();
        }
        // ---- epoch loss (hybrid_nn.cpp:190-192): trace[e] = sum r^2 / n ------
        LS[tid] = lossacc;
        lossacc = 0.0;
        __syncthreads();
        if (tid == 0 && p.trace) {
            double s = 0.0;
            for (int i = 0; i < kW8dThreads; ++i) s += LS[i];
            p.trace[(size_t)net * p.epochs + e] = s / (double)n;
        }
        __syncthreads();
    }
    // ---- trained parameters out (reference flat order) ---------------------
    for (int i = tid; i < 64 * IN; i += kW8dThreads) theta[i] = W[(i / IN) * G::WS + i % IN];
    if (tid < 64) {
        theta[64 * IN + tid] = B[tid];
        theta[64 * IN + 64 + tid] = F[tid];
    }
}

// widened FP64 rows [S][rows][width] from the complex design (iq_transform.cpp:17-20)
__global__ void widen64_kernel(const double *__restrict__ x, double *__restrict__ wide, size_t nrow_c, int m) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nrow_c * 2 * m) return;
    const size_t t = i / (2 * m);
    const int c = (int)(i % (2 * m));
    const double *xr = x + t * m * 2;
    const double re = c < m ? xr[2 * c] : xr[2 * (c - m)], im = c < m ? xr[2 * c + 1] : xr[2 * (c - m) + 1];
    wide[(2 * t) * 2 * m + c] = c < m ? re : im;
    wide[(2 * t + 1) * 2 * m + c] = c < m ? im : -re;
}

// 1 - beta_i^t for every step, FP64 pow (hybrid_nn.cpp:133-135)
__global__ void corr_table_kernel(double b1, double b2, int total, double *t) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < total) {
        t[2 * i] = 1.0 - pow(b1, (double)(i + 1));
        t[2 * i + 1] = 1.0 - pow(b2, (double)(i + 1));
    }
}

bool train_w8d_fits(const TrainF64Params &p) {
    const NetGeom &g = p.g;
    if (std::getenv("NOMA_TRAIN_W8D") && std::atoi(std::getenv("NOMA_TRAIN_W8D")) == 0) return false;
    return g.nd == 2 && g.dims[1] == 64 && (g.dims[0] == 32 || g.dims[0] == 64) && p.batch >= 1 &&
           p.batch <= kBatchRows && p.rows <= 65535;
}

int train_w8d_launch(TrainF64Params &p, cudaStream_t st) {
    const int IN = p.g.dims[0];
    const int total = p.epochs * ((p.rows + p.batch - 1) / p.batch);
    const double *wide = p.design;
    double *tmp = nullptr, *ctab = nullptr;
    const size_t nrow = (size_t)(p.n_nets / p.K) * p.rows;
    if (p.layout == NOMA_LAYOUT_WIDEN_COMPLEX) {
        if (cudaMallocAsync(&tmp, nrow * IN * sizeof(double), st) != cudaSuccess) return NOMA_ERR_CUDA;
        const size_t tot = (nrow / 2) * IN;
        widen64_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(p.design, tmp, nrow / 2, IN / 2);
        wide = tmp;
    }
    if (cudaMallocAsync(&ctab, 2 * (size_t)(total > 0 ? total : 1) * sizeof(double), st) != cudaSuccess) {
        if (tmp) cudaFreeAsync(tmp, st);
        return NOMA_ERR_CUDA;
    }
    if (total > 0) corr_table_kernel<<<(total + 255) / 256, 256, 0, st>>>(p.b1, p.b2, total, ctab);
    auto go = [&](auto kern, size_t smem) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<p.n_nets, kW8dThreads, smem, st>>>(p, wide, ctab);
    };
    if (IN == 32)
        go(train_w8d_kernel<32>, W8dGeom<32>::bytes);
    else
        go(train_w8d_kernel<64>, W8dGeom<64>::bytes);
    const int rc = cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;
    cudaFreeAsync(ctab, st);
    if (tmp) cudaFreeAsync(tmp, st);
    return rc;
}

}  // namespace noma_dev
