// Shape-general dense kernels of the detector: the paths the reference takes
// for networks outside the fused kernels' range and the FP64 entry points of
// its C++ API.
//
//  * fwd_tile_kernel<T>: single-pass forward of X w0 + a_N w_{N+1} over row
//    tiles, every layer's activations of the tile in shared memory
//    (feature-major [c][row]); the tile height adapts to the widest layer, so
//    any width up to ~25k fits.  FP64 instance = fused::fused_forward /
//    hybrid_nn::forward (fused_inference.cpp:62-127, hybrid_nn.cpp:60-82);
//    FP32 instance = fused_forward_f32 and the batched detection of networks
//    wider than 128 (decision + BER/SER epilogue, eval.cpp:38-65).
//  * layer_kernel<T> / lin_final_kernel<T>: per-layer evaluation with the
//    activations in HBM -- the reference's fallback_kernel (fused_inference.cpp:
//    132-151) and, with bias and ReLU as separate launches, its naive per-layer
//    path; also the forward half of loss_and_grad.
//  * rowdot / mask / outer / back kernels: hybrid_nn::loss_and_grad
//    (hybrid_nn.cpp:84-114) in FP64, deterministic fixed-order reductions.
//  * adam_kernel: hybrid_nn::adam_step (hybrid_nn.cpp:118-144) in FP64 with the
//    reference's operation order and no FMA contraction.
//
// The linear branch x.w0 is accumulated from 0 in column order with separate
// multiply and add, like the reference's column-major GEMV built with
// -ffp-contract=off (CMakeLists.txt:27), so a zero final layer reproduces
// X w0 bit for bit (test_hybrid_nn.cpp:44-53, test_fused.cpp:76-85).
#include <math.h>

#include <algorithm>

#include "kernels.cuh"

namespace noma_dev {

template <class T>
__device__ __forceinline__ T mul_rn(T a, T b);
template <>
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
template <>
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
template <class T>
__device__ __forceinline__ T add_rn(T a, T b);
template <>
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
template <>
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }

// ------------------------------------------------------ single-pass forward
template <class T>
__device__ __forceinline__ T load_in(const FwdParams<T> &p, int d, int R, int c) {
    // widened / real input row R, column c of design d
    if (p.src == kSrcColMajor) return p.x[(size_t)c * p.ldx + R];
    if (p.src == kSrcRowMajor) return p.x[((size_t)d * p.stride + R) * p.g.dims[0] + c];
    const int m = p.g.dims[0] / 2, t = R >> 1;  // complex rows: iq_transform.cpp:17-20
    const T *xr = p.x + ((size_t)d * p.stride + t) * m * 2;
    if (c < m) return (R & 1) ? xr[2 * c + 1] : xr[2 * c];
    return (R & 1) ? -xr[2 * (c - m)] : xr[2 * (c - m) + 1];
}

template <class T>
__global__ void __launch_bounds__(256) fwd_tile_kernel(FwdParams<T> p) {
    extern __shared__ __align__(16) unsigned char fwd_smem[];
    T *sm = reinterpret_cast<T *>(fwd_smem);
    const NetGeom &g = p.g;
    const int net = blockIdx.y, d = net / p.K, TR = p.TR, tid = threadIdx.x, nt = blockDim.x;
    if (p.status && p.status[net] != NOMA_OK) {
        if (blockIdx.x == 0 && tid == 0) {
            if (p.errors) p.errors[net] = 0xFFFFFFFFu;
            if (p.sym_errors) p.sym_errors[net] = 0xFFFFFFFFu;
        }
        return;
    }
    const int r0 = blockIdx.x * TR, nr = min(TR, p.rows - r0);
    if (nr <= 0) return;
    const T *plan = p.plan + (size_t)net * g.plan_total;
    const int d0 = g.dims[0];
    T *A0 = sm;                        // input tile [d0][TR]
    T *A1 = A0 + (size_t)d0 * TR;      // hidden ping [maxh][TR]
    T *A2 = A1 + (size_t)p.maxh * TR;  // hidden pong
    T *Y = A2 + (size_t)p.maxh * TR;   // outputs [TR]
    for (int i = tid; i < d0 * TR; i += nt) {
        const int c = i / TR, r = i - c * TR;
        A0[i] = r < nr ? load_in(p, d, r0 + r, c) : T(0);
    }
    __syncthreads();
    const T *in = A0;
    T *out = A1;
    for (int l = 1; l < g.nd; ++l) {
        const int din = g.dims[l - 1], dout = g.dims[l], ws = g.plan_pad[l - 1];
        const T *W = plan + g.plan_w[l], *b = plan + g.plan_b[l];
        for (int i = tid; i < dout * TR; i += nt) {
            const int j = i / TR, r = i - j * TR;
            const T *wj = W + (size_t)j * ws;
            T acc = b[j];
            for (int c = 0; c < din; ++c) acc = fma(wj[c], in[c * TR + r], acc);
            out[i] = acc > T(0) ? acc : T(0);
        }
        __syncthreads();
        in = out;
        out = out == A1 ? A2 : A1;
    }
    const int dN = g.dims[g.nd - 1];
    const T *w0 = plan + g.plan_w0, *wf = plan + g.plan_f;
    for (int r = tid; r < nr; r += nt) {
        T lin = T(0), br = T(0);
        for (int c = 0; c < d0; ++c) lin = add_rn(lin, mul_rn(A0[c * TR + r], w0[c]));
        for (int j = 0; j < dN; ++j) br = add_rn(br, mul_rn(in[j * TR + r], wf[j]));
        Y[r] = add_rn(lin, br);
    }
    __syncthreads();
    if (p.out)
        for (int r = tid; r < nr; r += nt) p.out[(size_t)net * p.out_stride + r0 + r] = Y[r];
    if (p.src != kSrcComplex) return;
    // QPSK decision of each symbol (row pair) and the BER/SER counters
    // (eval.cpp:38-65): bit0 = Re < 0, bit1 = Im < 0
    const int npair = nr / 2;
    unsigned be = 0, se = 0;
    for (int q = tid; q < npair; q += nt) {
        const int t = (r0 >> 1) + q;
        const uint8_t code = (uint8_t)((Y[2 * q] < T(0) ? 1 : 0) | (Y[2 * q + 1] < T(0) ? 2 : 0));
        if (p.codes) p.codes[(size_t)net * p.code_stride + t] = code;
        if (p.truth) {
            const uint8_t tr = p.truth[((size_t)d * p.stride + t) * p.K + (net - d * p.K)];
            be += __popc((unsigned)(code ^ tr));
            se += code != tr;
        }
    }
    if (p.truth && (p.errors || p.sym_errors)) {
        be = __reduce_add_sync(0xffffffffu, be);
        se = __reduce_add_sync(0xffffffffu, se);
        if ((tid & 31) == 0 && (be || se)) {
            if (p.errors && be) atomicAdd(p.errors + net, be);
            if (p.sym_errors && se) atomicAdd(p.sym_errors + net, se);
        }
    }
}

template <class T>
int fwd_tile_launch(FwdParams<T> &p, cudaStream_t st) {
    const NetGeom &g = p.g;
    int maxh = 1;
    for (int l = 1; l < g.nd; ++l) maxh = g.dims[l] > maxh ? g.dims[l] : maxh;
    p.maxh = maxh;
    const size_t per_row = ((size_t)g.dims[0] + 2 * (size_t)maxh + 1) * sizeof(T);
    const size_t budget = 200 * 1024;
    int TR = (int)std::min<size_t>(64, budget / per_row);
    TR &= ~1;  // whole symbols (row pairs) per tile
    if (TR < 2) return NOMA_ERR_UNSUPPORTED;
    p.TR = TR;
    if (p.rows <= 0 || p.n_nets <= 0) return NOMA_OK;
    const size_t smem = per_row * TR;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(fwd_tile_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return NOMA_ERR_CUDA;
    const dim3 grid((p.rows + TR - 1) / TR, p.n_nets);
    if (grid.y > 65535) return NOMA_ERR_UNSUPPORTED;
    fwd_tile_kernel<T><<<grid, 256, smem, st>>>(p);
    return cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;
}
template int fwd_tile_launch<float>(FwdParams<float> &, cudaStream_t);
template int fwd_tile_launch<double>(FwdParams<double> &, cudaStream_t);

// ------------------------------------------------------ per-layer kernels
// Activations feature-major in HBM: A[c * ld + r].
template <class T>
__global__ void layer_kernel(const T *A, long long lda, int din, const T *W, int wstride, const T *b, int dout,
                             T *Z, long long ldz, int rows, int relu) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
    if (r >= rows || j >= dout) return;
    const T *wj = W + (size_t)j * wstride;
    T acc = b ? b[j] : T(0);
    for (int c = 0; c < din; ++c) acc = fma(wj[c], A[(size_t)c * lda + r], acc);
    Z[(size_t)j * ldz + r] = relu ? (acc > T(0) ? acc : T(0)) : acc;
}

template <class T>
__global__ void bias_relu_kernel(T *Z, long long ldz, const T *b, int dout, int rows, int mode) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
    if (r >= rows || j >= dout) return;
    T &z = Z[(size_t)j * ldz + r];
    if (mode == 0) z = z + b[j];
    else z = z > T(0) ? z : T(0);
}

// y[r] = x_r.w0 + a_r.w_f (fallback / naive output), or with targets the
// residual x_r.w0 + a_r.w_f - y_r (hybrid_nn.cpp:94) and dy = (2/B) r (:98)
template <class T>
__global__ void lin_final_kernel(const T *X, long long ldx, int d0, const T *w0, const T *AN, long long ldan, int dN,
                                 const T *wf, int rows, const T *y, T *out, T *dy, T two_over_b) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    T lin = T(0), br = T(0);
    for (int c = 0; c < d0; ++c) lin = add_rn(lin, mul_rn(X[(size_t)c * ldx + r], w0[c]));
    for (int j = 0; j < dN; ++j) br = add_rn(br, mul_rn(AN[(size_t)j * ldan + r], wf[j]));
    T v = add_rn(lin, br);
    if (y) {
        v = v - y[r];
        if (dy) dy[r] = mul_rn(two_over_b, v);
    }
    out[r] = v;
}

// out[i * nq + q] = sum_b P[i * ldp + b] * Q[q * ldq + b] (Q null: row sums),
// one warp per output, lanes strided over b, fixed-order xor tree
template <class T>
__global__ void rowdot_kernel(const T *P, long long ldp, const T *Q, long long ldq, int ni, int nq, int len, T *out) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= ni * nq) return;
    const int i = w / nq, q = w - i * nq;
    const T *pi = P + (size_t)i * ldp;
    const T *qq = Q ? Q + (size_t)q * ldq : nullptr;
    T acc = T(0);
    for (int b = lane; b < len; b += 32) acc = qq ? fma(pi[b], qq[b], acc) : acc + pi[b];
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[w] = acc;
}

// dA_N[j][r] = dy[r] * w_f[j] (hybrid_nn.cpp:102)
template <class T>
__global__ void outer_kernel(const T *dy, const T *wf, int dN, int rows, T *dA, long long ld) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
    if (r >= rows || j >= dN) return;
    dA[(size_t)j * ld + r] = dy[r] * wf[j];
}

// dz = (a_n > 0) ? da : 0 (hybrid_nn.cpp:107), in place
template <class T>
__global__ void mask_kernel(const T *A, T *D, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && !(A[i] > T(0))) D[i] = T(0);
}

// da_{n-1}[c][r] = sum_j dz[j][r] W_n[j][c] (hybrid_nn.cpp:111)
template <class T>
__global__ void back_kernel(const T *W, int wstride, int din, int dout, const T *dZ, long long ld, int rows, T *dA) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x, c = blockIdx.y;
    if (r >= rows || c >= din) return;
    T acc = T(0);
    for (int j = 0; j < dout; ++j) acc = fma(dZ[(size_t)j * ld + r], W[(size_t)j * wstride + c], acc);
    dA[(size_t)c * ld + r] = acc;
}

// loss = ||r||^2 / B, one CTA, fixed-order tree
template <class T>
__global__ void sqnorm_kernel(const T *r, int n, T inv_b, T *loss) {
    __shared__ T red[256];
    T acc = T(0);
    for (int i = threadIdx.x; i < n; i += 256) acc = fma(r[i], r[i], acc);
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = 128; s; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) *loss = red[0] * inv_b;
}

// Adam (hybrid_nn.cpp:118-124): m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2;
// theta -= lr (m / c1) / (sqrt(v / c2) + eps), c_i = 1 - beta_i^step from the
// host's std::pow; rounded operation by operation like the reference build.
__global__ void adam_kernel(int n, double *theta, const double *grad, double *m, double *v, double c1, double c2,
                            double lr, double b1, double b2, double eps) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double g = grad[i];
    const double mi = __dadd_rn(__dmul_rn(b1, m[i]), __dmul_rn(__dsub_rn(1.0, b1), g));
    const double vi = __dadd_rn(__dmul_rn(b2, v[i]), __dmul_rn(__dsub_rn(1.0, b2), __dmul_rn(g, g)));
    m[i] = mi;
    v[i] = vi;
    const double num = __dmul_rn(lr, __ddiv_rn(mi, c1));
    const double den = __dadd_rn(__dsqrt_rn(__ddiv_rn(vi, c2)), eps);
    theta[i] = __dsub_rn(theta[i], __ddiv_rn(num, den));
}

// ------------------------------------------------------ launchers
namespace {
inline dim3 rows_grid(int rows, int y) { return dim3((rows + 127) / 128, y); }
inline bool ok() { return cudaGetLastError() == cudaSuccess; }
}  // namespace

// Per-layer forward of one network (plan layout), X feature-major [d0][ld];
// acts: scratch holding every layer's activations [sum dims[1..]][ld]
// (layer l at acts + act_off(l)).  naive: GEMM, bias and ReLU as three
// launches per layer.  With y: residual + dy instead of the output.
template <class T>
int layer_forward_launch(const NetGeom &g, const T *plan, const T *X, long long ld, int rows, T *acts, bool naive,
                         const T *y, T *out, T *dy, cudaStream_t st) {
    if (rows <= 0) return NOMA_OK;
    const T *in = X;
    long long off = 0;
    for (int l = 1; l < g.nd; ++l) {
        T *Z = acts + off * ld;
        const T *W = plan + g.plan_w[l], *b = plan + g.plan_b[l];
        if (naive) {
            layer_kernel<T><<<rows_grid(rows, g.dims[l]), 128, 0, st>>>(in, ld, g.dims[l - 1], W, g.plan_pad[l - 1],
                                                                        nullptr, g.dims[l], Z, ld, rows, 0);
            bias_relu_kernel<T><<<rows_grid(rows, g.dims[l]), 128, 0, st>>>(Z, ld, b, g.dims[l], rows, 0);
            bias_relu_kernel<T><<<rows_grid(rows, g.dims[l]), 128, 0, st>>>(Z, ld, b, g.dims[l], rows, 1);
        } else {
            layer_kernel<T><<<rows_grid(rows, g.dims[l]), 128, 0, st>>>(in, ld, g.dims[l - 1], W, g.plan_pad[l - 1], b,
                                                                        g.dims[l], Z, ld, rows, 1);
        }
        in = Z;
        off += g.dims[l];
    }
    lin_final_kernel<T><<<(rows + 127) / 128, 128, 0, st>>>(X, ld, g.dims[0], plan + g.plan_w0, in, ld,
                                                            g.dims[g.nd - 1], plan + g.plan_f, rows, y, out, dy,
                                                            T(2) / T(rows));
    return ok() ? NOMA_OK : NOMA_ERR_CUDA;
}
template int layer_forward_launch<float>(const NetGeom &, const float *, const float *, long long, int, float *, bool,
                                         const float *, float *, float *, cudaStream_t);
template int layer_forward_launch<double>(const NetGeom &, const double *, const double *, long long, int, double *,
                                          bool, const double *, double *, double *, cudaStream_t);

// hybrid_nn::loss_and_grad (hybrid_nn.cpp:84-114) for one network in FP64.
// ws: >= loss_grad_scratch(g, rows) doubles.  grad: flat reference order
// (W_1 row-major, b_1, ..., W_N, b_N, final).
size_t loss_grad_scratch(const NetGeom &g, int rows) {
    size_t h = 0;
    int maxw = g.dims[0];
    for (int l = 1; l < g.nd; ++l) {
        h += g.dims[l];
        maxw = g.dims[l] > maxw ? g.dims[l] : maxw;
    }
    return (h + 2 * (size_t)maxw + 2) * (size_t)rows + 1;
}

int loss_grad_launch(const NetGeom &g, const double *plan, const double *X, int rows, const double *y, double *ws,
                     double *loss, double *grad, cudaStream_t st) {
    int maxw = g.dims[0];
    size_t h = 0;
    for (int l = 1; l < g.nd; ++l) {
        h += g.dims[l];
        maxw = g.dims[l] > maxw ? g.dims[l] : maxw;
    }
    const long long ld = rows;
    double *acts = ws, *dA = acts + h * ld, *dB = dA + (size_t)maxw * ld, *res = dB + (size_t)maxw * ld,
           *dy = res + ld;
    int st_ = layer_forward_launch<double>(g, plan, X, ld, rows, acts, false, y, res, dy, st);
    if (st_) return st_;
    sqnorm_kernel<double><<<1, 256, 0, st>>>(res, rows, 1.0 / rows, loss);
    // activation offsets
    size_t aoff[NOMA_MAX_DIMS];
    size_t o = 0;
    for (int l = 1; l < g.nd; ++l) {
        aoff[l] = o;
        o += g.dims[l];
    }
    auto act = [&](int l) -> const double * { return l == 0 ? X : acts + aoff[l] * ld; };
    // grad offsets (flat reference order)
    size_t gw[NOMA_MAX_DIMS], gb[NOMA_MAX_DIMS];
    o = 0;
    for (int l = 1; l < g.nd; ++l) {
        gw[l] = o;
        o += (size_t)g.dims[l] * g.dims[l - 1];
        gb[l] = o;
        o += g.dims[l];
    }
    const size_t gf = o;
    const int N = g.nd - 1, dN = g.dims[N];
    // g_final = a_N^T dy (:99)
    rowdot_kernel<double><<<(dN * 32 + 255) / 256, 256, 0, st>>>(act(N), ld, dy, ld, dN, 1, rows, grad + gf);
    if (N == 0) return ok() ? NOMA_OK : NOMA_ERR_CUDA;
    outer_kernel<double><<<rows_grid(rows, dN), 128, 0, st>>>(dy, plan + g.plan_f, dN, rows, dA, ld);
    for (int n = N; n >= 1; --n) {
        const int dout = g.dims[n], din = g.dims[n - 1];
        mask_kernel<double><<<(unsigned)(((size_t)dout * ld + 255) / 256), 256, 0, st>>>(act(n), dA, (long long)dout * ld);
        rowdot_kernel<double><<<(unsigned)(((size_t)dout * din * 32 + 255) / 256), 256, 0, st>>>(
            dA, ld, act(n - 1), ld, dout, din, rows, grad + gw[n]);
        rowdot_kernel<double><<<(dout * 32 + 255) / 256, 256, 0, st>>>(dA, ld, nullptr, 0, dout, 1, rows, grad + gb[n]);
        if (n > 1) {
            back_kernel<double><<<rows_grid(rows, din), 128, 0, st>>>(plan + g.plan_w[n], g.plan_pad[n - 1], din, dout,
                                                                     dA, ld, rows, dB);
            double *t = dA;
            dA = dB;
            dB = t;
        }
    }
    return ok() ? NOMA_OK : NOMA_ERR_CUDA;
}

int adam_launch(int n, double *theta, const double *grad, double *m, double *v, double c1, double c2, double lr,
                double b1, double b2, double eps, cudaStream_t st) {
    if (n <= 0) return NOMA_OK;
    adam_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, theta, grad, m, v, c1, c2, lr, b1, b2, eps);
    return ok() ? NOMA_OK : NOMA_ERR_CUDA;
}

}  // namespace noma_dev
