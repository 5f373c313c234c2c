// Shape-general pilot-phase training (hybrid_nn::train, hybrid_nn.cpp:158-195
// with loss_and_grad :84-114 and adam_step :118-144) for the networks the
// on-chip kernels do not cover: layers wider than 128, minibatches above 128
// rows, or FP64 nets too large for k_train_f64's shared-memory layout.
//
// One CTA per user network runs every epoch and minibatch in one launch.  The
// parameters are trained in place in their FusedPlan layout (the reference's
// packed buffer, fused_inference.cpp:19-42); gradients, Adam moments and the
// minibatch's activations live in a per-net HBM/L2 scratch, feature-major
// ([feature][row]) so every phase reads rows contiguously.  Reductions over
// the minibatch are one warp per output with a fixed xor tree, so repeated
// runs are bit-identical (test_hybrid_nn.cpp:290-311).
//
// T = float: the batch kernels' precision (FP32 design rows and the FP64
// residual r0 = y - X w0 rounded to FP32, the frozen branch folded out).
// T = double: the reference's precision, residual x w0 + a_N w - y formed as
// hybrid_nn.cpp:94 does.
#include <math.h>

#include "kernels.cuh"

namespace noma_dev {

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <class T>
__global__ void __launch_bounds__(256) train_generic_kernel(TrainGenParams<T> p) {
    __shared__ double red[8];
    __shared__ T corr[2];
    const int net = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (p.status && p.status[net] != NOMA_OK) return;
    const NetGeom &g = p.g;
    const int N = g.nd - 1, n = p.rows, d = net / p.K, B = p.batch, d0 = g.dims[0], dN = g.dims[N];
    T *plan = p.plan + (size_t)net * g.plan_total;
    T *ws = p.scratch + (size_t)net * p.scratch_per_net;
    T *G = ws, *Mo = G + g.plan_total, *Vo = Mo + g.plan_total;
    T *XB = Vo + g.plan_total;
    T *ACT = XB + (size_t)d0 * B;
    size_t aoff[NOMA_MAX_DIMS] = {0};
    for (int l = 2; l <= N; ++l) aoff[l] = aoff[l - 1] + g.dims[l - 1];
    size_t hsum = 0;
    int maxw = d0;
    for (int l = 1; l <= N; ++l) {
        hsum += g.dims[l];
        maxw = g.dims[l] > maxw ? g.dims[l] : maxw;
    }
    T *DA = ACT + hsum * B, *DB = DA + (size_t)maxw * B, *RB = DB + (size_t)maxw * B, *DY = RB + B, *YB = DY + B;
    auto act = [&](int l) -> T * { return l == 0 ? XB : ACT + aoff[l] * B; };
    for (int i = tid; i < 3 * g.plan_total; i += 256) G[i] = T(0);  // grads (pads stay 0) and moments
    const uint16_t *perm_net = p.perm + (size_t)net * p.epochs * n;
    const double *w0d = p.w0 ? p.w0 + (size_t)net * d0 : nullptr;
    long long step = 0;
    __syncthreads();
    for (int e = 0; e < p.epochs; ++e) {
        const uint16_t *perm = perm_net + (size_t)e * n;
        double loss_sum = 0.0;
        for (int start = 0; start < n; start += B) {
            const int b = min(B, n - start);
            // gather the permuted minibatch, IQ widening at load (iq_transform.cpp:17-20)
            for (int i = tid; i < d0 * b; i += 256) {
                const int c = i / b, r = i - c * b, row = perm[start + r];
                T v;
                if constexpr (sizeof(T) == 4) {
                    if (p.layout == NOMA_LAYOUT_WIDEN_COMPLEX) {
                        const float *xr = p.design32 + ((size_t)d * (n / 2) + (row >> 1)) * d0;
                        const int m = d0 / 2;
                        v = (row & 1) ? (c < m ? xr[m + c] : -xr[c - m]) : xr[c];
                    } else {
                        v = p.design32[((size_t)d * n + row) * d0 + c];
                    }
                } else {
                    if (p.layout == NOMA_LAYOUT_WIDEN_COMPLEX) {
                        const int m = d0 / 2;
                        const double *xr = p.design + ((size_t)d * (n / 2) + (row >> 1)) * m * 2;
                        if (c < m) v = (row & 1) ? xr[2 * c + 1] : xr[2 * c];
                        else v = (row & 1) ? -xr[2 * (c - m)] : xr[2 * (c - m) + 1];
                    } else {
                        v = p.design[((size_t)d * n + row) * d0 + c];
                    }
                }
                XB[(size_t)c * B + r] = v;
            }
            for (int r = tid; r < b; r += 256) {
                const int row = perm[start + r];
                if constexpr (sizeof(T) == 4) {
                    YB[r] = p.r0[(size_t)net * n + row];
                } else {
                    // targets: WIDEN [S][rows/2][K] complex = interleaved per
                    // (t, k); REAL [S][K][rows]
                    const int k = net - d * p.K;
                    YB[r] = p.layout == NOMA_LAYOUT_WIDEN_COMPLEX
                                ? p.targets[(((size_t)d * (n / 2) + (row >> 1)) * p.K + k) * 2 + (row & 1)]
                                : p.targets[((size_t)d * p.K + k) * n + row];
                }
            }
            __syncthreads();
            // forward: a_l = max(a_{l-1} W_l^T + b_l, 0) (hybrid_nn.cpp:60-70)
            for (int l = 1; l <= N; ++l) {
                const int din = g.dims[l - 1], dout = g.dims[l], ws_ = g.plan_pad[l - 1];
                const T *W = plan + g.plan_w[l], *bb = plan + g.plan_b[l];
                const T *in = act(l - 1);
                T *out = act(l);
                for (int i = tid; i < dout * b; i += 256) {
                    const int j = i / b, r = i - j * b;
                    const T *wj = W + (size_t)j * ws_;
                    T acc = bb[j];
                    for (int c = 0; c < din; ++c) acc = fma(wj[c], in[(size_t)c * B + r], acc);
                    out[(size_t)j * B + r] = acc > T(0) ? acc : T(0);
                }
                __syncthreads();
            }
            // residual and dy = (2/b) r (hybrid_nn.cpp:94-98)
            const T two_b = T(2) / T(b);
            double part = 0.0;
            {
                const T *AN = act(N), *wf = plan + g.plan_f;
                for (int r = tid; r < b; r += 256) {
                    T br = T(0);
                    for (int j = 0; j < dN; ++j) br = fma(AN[(size_t)j * B + r], wf[j], br);
                    T res;
                    if constexpr (sizeof(T) == 4) {
                        res = br - YB[r];
                    } else {
                        double lin = 0.0;
                        for (int c = 0; c < d0; ++c) lin = __dadd_rn(lin, __dmul_rn(XB[(size_t)c * B + r], w0d[c]));
                        res = (lin + br) - YB[r];
                    }
                    RB[r] = res;
                    DY[r] = two_b * res;
                    part += (double)res * (double)res;
                }
            }
            part = warp_sum(part);
            if (lane == 0) red[warp] = part;
            __syncthreads();
            if (tid == 0) {
                double s = 0.0;
                for (int w = 0; w < 8; ++w) s += red[w];
                loss_sum += (s / b) * b;  // loss_b * b (hybrid_nn.cpp:190)
            }
            // g_final = a_N^T dy, dA_N = dy w_f^T (:99-102)
            {
                const T *AN = act(N), *wf = plan + g.plan_f;
                for (int j = warp; j < dN; j += 8) {
                    T acc = T(0);
                    for (int r = lane; r < b; r += 32) acc = fma(AN[(size_t)j * B + r], DY[r], acc);
                    acc = warp_sum(acc);
                    if (lane == 0) G[g.plan_f + j] = acc;
                }
                if (N > 0)
                    for (int i = tid; i < dN * b; i += 256) {
                        const int j = i / b, r = i - j * b;
                        DA[(size_t)j * B + r] = DY[r] * wf[j];
                    }
            }
            __syncthreads();
            T *da = DA, *db = DB;
            for (int l = N; l >= 1; --l) {
                const int dout = g.dims[l], din = g.dims[l - 1], ws_ = g.plan_pad[l - 1];
                const T *A = act(l), *Ab = act(l - 1), *W = plan + g.plan_w[l];
                for (int i = tid; i < dout * b; i += 256) {  // dz = (a_l > 0) ? da : 0 (:107)
                    const int j = i / b, r = i - j * b;
                    if (!(A[(size_t)j * B + r] > T(0))) da[(size_t)j * B + r] = T(0);
                }
                __syncthreads();
                // gW = dz^T a_{l-1}, gb = colsum dz (:109-110)
                for (int o = warp; o < dout * (din + 1); o += 8) {
                    const int j = o / (din + 1), c = o - j * (din + 1);
                    T acc = T(0);
                    if (c < din)
                        for (int r = lane; r < b; r += 32) acc = fma(da[(size_t)j * B + r], Ab[(size_t)c * B + r], acc);
                    else
                        for (int r = lane; r < b; r += 32) acc += da[(size_t)j * B + r];
                    acc = warp_sum(acc);
                    if (lane == 0) G[c < din ? g.plan_w[l] + (size_t)j * ws_ + c : g.plan_b[l] + j] = acc;
                }
                if (l > 1)  // da_{l-1} = dz W_l (:111)
                    for (int i = tid; i < din * b; i += 256) {
                        const int c = i / b, r = i - c * b;
                        T acc = T(0);
                        for (int j = 0; j < dout; ++j) acc = fma(da[(size_t)j * B + r], W[(size_t)j * ws_ + c], acc);
                        db[(size_t)c * B + r] = acc;
                    }
                __syncthreads();
                T *t = da;
                da = db;
                db = t;
            }
            // Adam (hybrid_nn.cpp:129-143): corrections from FP64 pow, every
            // trainable entry of the plan (w0 excluded; pads have zero
            // gradient and stay zero)
            ++step;
            if (tid == 0) {
                corr[0] = (T)(1.0 - pow(p.b1, (double)step));
                corr[1] = (T)(1.0 - pow(p.b2, (double)step));
            }
            __syncthreads();
            const T c1 = corr[0], c2 = corr[1], lr = (T)p.lr, b1 = (T)p.b1, b2 = (T)p.b2, eps = (T)p.eps;
            for (int i = g.plan_pad[0] + tid; i < g.plan_total; i += 256) {
                const T gr = G[i];
                const T m = b1 * Mo[i] + (T(1) - b1) * gr;
                const T v = b2 * Vo[i] + (T(1) - b2) * (gr * gr);
                Mo[i] = m;
                Vo[i] = v;
                plan[i] -= lr * (m / c1) / (sqrt(v / c2) + eps);
            }
            __syncthreads();
        }
        if (tid == 0 && p.trace) p.trace[(size_t)net * p.epochs + e] = loss_sum / n;
    }
}

size_t train_generic_scratch(const NetGeom &g, int batch) {
    size_t hsum = 0;
    int maxw = g.dims[0];
    for (int l = 1; l < g.nd; ++l) {
        hsum += g.dims[l];
        maxw = g.dims[l] > maxw ? g.dims[l] : maxw;
    }
    return 3 * (size_t)g.plan_total + ((size_t)g.dims[0] + hsum + 2 * (size_t)maxw + 3) * batch;
}

template <class T>
int train_generic_launch(TrainGenParams<T> &p, cudaStream_t st) {
    if (p.n_nets <= 0 || p.epochs <= 0) return NOMA_OK;
    if (p.batch < 1 || p.rows > 65535) return NOMA_ERR_UNSUPPORTED;
    train_generic_kernel<T><<<p.n_nets, 256, 0, st>>>(p);
    return cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;
}
template int train_generic_launch<float>(TrainGenParams<float> &, cudaStream_t);
template int train_generic_launch<double>(TrainGenParams<double> &, cudaStream_t);

// theta (flat reference order: W_1 row-major, b_1, ..., W_N, b_N, final;
// hybrid_nn.hpp:15-23) <-> FusedPlan layout (fused_inference.cpp:19-42).
// to_plan: plan = [w0 | W_l rows padded, b_l | final], pads zero.
__global__ void theta_plan_kernel(NetGeom g, int n_nets, int ptrain, double *theta, double *plan, const double *w0,
                                  int to_plan) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)n_nets * g.plan_total) return;
    const int net = (int)(i / g.plan_total), q = (int)(i - (size_t)net * g.plan_total);
    double *th = theta + (size_t)net * ptrain;
    double *pl = plan + (size_t)net * g.plan_total;
    int t = -1;  // flat theta index of plan entry q (-1: w0 slot or pad)
    if (q >= g.plan_f) {
        const int j = q - g.plan_f;
        if (j < g.dims[g.nd - 1]) {
            int o = 0;
            for (int l = 1; l < g.nd; ++l) o += g.dims[l] * g.dims[l - 1] + g.dims[l];
            t = o + j;
        }
    } else if (q >= g.plan_pad[0]) {
        int o = 0;
        for (int l = 1; l < g.nd; ++l) {
            if (q >= g.plan_w[l] && q < g.plan_b[l]) {
                const int j = (q - g.plan_w[l]) / g.plan_pad[l - 1], c = (q - g.plan_w[l]) - j * g.plan_pad[l - 1];
                if (c < g.dims[l - 1]) t = o + j * g.dims[l - 1] + c;
                break;
            }
            o += g.dims[l] * g.dims[l - 1];
            if (q >= g.plan_b[l] && q < g.plan_b[l] + g.plan_pad[l]) {
                const int j = q - g.plan_b[l];
                if (j < g.dims[l]) t = o + j;
                break;
            }
            o += g.dims[l];
        }
    }
    if (to_plan) {
        if (q < g.plan_pad[0]) pl[q] = (w0 && q < g.dims[0]) ? w0[(size_t)net * g.dims[0] + q] : 0.0;
        else pl[q] = t >= 0 ? th[t] : 0.0;
    } else if (t >= 0) {
        th[t] = pl[q];
    }
}

int theta_plan_launch(const NetGeom &g, int n_nets, double *theta, double *plan, const double *w0, int to_plan,
                      cudaStream_t st) {
    const size_t n = (size_t)n_nets * g.plan_total;
    if (n == 0) return NOMA_OK;
    theta_plan_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(g, n_nets, trainable_count(g), theta, plan, w0,
                                                                  to_plan);
    return cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;
}

// FP64 theta (flat reference order) -> FP32 FusedPlan with w0 in its slot:
// the detection parameters of an FP64-trained net
__global__ void theta_plan32_kernel(NetGeom g, int n_nets, int ptrain, const double *theta, float *plan,
                                    const double *w0) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)n_nets * ptrain + (size_t)n_nets * g.dims[0]) return;
    if (i >= (size_t)n_nets * ptrain) {  // w0 slots
        const size_t k = i - (size_t)n_nets * ptrain;
        const int net = (int)(k / g.dims[0]), c = (int)(k - (size_t)net * g.dims[0]);
        plan[(size_t)net * g.plan_total + c] = (float)w0[k];
        return;
    }
    const int net = (int)(i / ptrain), t = (int)(i - (size_t)net * ptrain);
    int o = 0, q = -1;
    for (int l = 1; l < g.nd && q < 0; ++l) {
        const int nw = g.dims[l] * g.dims[l - 1];
        if (t < o + nw) {
            const int j = (t - o) / g.dims[l - 1], c = (t - o) - j * g.dims[l - 1];
            q = g.plan_w[l] + j * g.plan_pad[l - 1] + c;
        } else if (t < o + nw + g.dims[l]) {
            q = g.plan_b[l] + (t - o - nw);
        }
        o += nw + g.dims[l];
    }
    if (q < 0) q = g.plan_f + (t - o);
    plan[(size_t)net * g.plan_total + q] = (float)theta[i];
}

int theta_plan32_launch(const NetGeom &g, int n_nets, const double *theta, float *plan, const double *w0,
                        cudaStream_t st) {
    const int ptrain = trainable_count(g);
    const size_t n = (size_t)n_nets * (ptrain + g.dims[0]);
    if (n == 0) return NOMA_OK;
    cudaMemsetAsync(plan, 0, (size_t)n_nets * g.plan_total * sizeof(float), st);
    theta_plan32_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(g, n_nets, ptrain, theta, plan, w0);
    return cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;
}

}  // namespace noma_dev
