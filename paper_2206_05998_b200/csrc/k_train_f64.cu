// FP64 parity mode of the pilot-phase training (hybrid_nn::train,
// hybrid_nn.cpp:158-195, with loss_and_grad :84-114 and adam_step :118-144)
// -- the reference's own precision.  Same fused structure as the FP32 kernel
// (one CTA per user network for all epochs, weights/gradients on chip, the
// IQ widening applied at load) but every value is FP64 and the residual is
// formed exactly as the reference does (x w0 + a_N w - y, hybrid_nn.cpp:94).
// Used to show that the device path reproduces the FP64 reference trajectory;
// the FP32 kernel is the throughput path.
//
// The 128-row minibatch is processed in chunks of CH rows (CH = 64 or 32 so
// the FP64 activations fit next to the FP64 weights and gradients); gradients
// accumulate over the chunks before the single Adam update of the step.  Adam
// moments live in global memory (L2-resident), two FP64 per parameter.
#include <math.h>

#include "kernels.cuh"

namespace noma_dev {

constexpr int kT64 = 256;

__global__ void __launch_bounds__(kT64) train_f64_kernel(TrainF64Params p) {
    extern __shared__ __align__(16) double smd[];
    const int net = blockIdx.x, tid = threadIdx.x;
    if (p.status && p.status[net] != NOMA_OK) return;
    const NetGeom &g = p.g;
    const int N = g.nd - 1, n = p.rows, d = net / p.K, CH = p.chunk;
    const int width = p.width, M = width / 2;
    // theta layout (reference flat order): W_1 (L1 x L0), b_1, ..., final
    double *TH = smd;                      // ptrain
    double *GR = TH + p.ptrain;            // ptrain
    double *ACT = GR + p.ptrain;           // activations [layer][CH][L_l], layer 0 = input
    double *DA = ACT + p.act_total;        // dA scratch [CH][maxw]
    double *DZ = DA + CH * p.maxw;         // dZ scratch [CH][maxw]
    double *YB = DZ + CH * p.maxw;         // targets of the chunk [CH]
    double *RED = YB + CH;                 // kT64 reduction scratch
    int *IDX = reinterpret_cast<int *>(RED + kT64);  // CH row indices

    double *gtheta = p.theta + (size_t)net * p.ptrain;
    double *m1 = p.moments + (size_t)net * 2 * p.ptrain, *m2 = m1 + p.ptrain;
    for (int i = tid; i < p.ptrain; i += kT64) {
        TH[i] = gtheta[i];
        m1[i] = 0.0;
        m2[i] = 0.0;
    }
    const double *w0 = p.w0 + (size_t)net * width;
    int woff[NOMA_MAX_DIMS], boff[NOMA_MAX_DIMS], aoff[NOMA_MAX_DIMS];
    {
        int o = 0, a = 0;
        for (int l = 1; l <= N; ++l) {
            woff[l] = o;
            o += g.dims[l] * g.dims[l - 1];
            boff[l] = o;
            o += g.dims[l];
        }
        for (int l = 0; l <= N; ++l) {  // activation rows padded by one double (banks)
            aoff[l] = a;
            a += CH * (g.dims[l] + 1);
        }
    }
    const int foff = p.ptrain - g.dims[N];
    __syncthreads();
    long step = 0;
    for (int e = 0; e < p.epochs; ++e) {
        const uint16_t *perm = p.perm + ((size_t)net * p.epochs + e) * n;
        double loss_sum = 0.0;  // thread 0
        for (int start = 0; start < n; start += p.batch) {
            const int bsz = min(p.batch, n - start);
            for (int i = tid; i < p.ptrain; i += kT64) GR[i] = 0.0;
            double sq = 0.0;  // per-thread partial of ||residual||^2
            __syncthreads();
            for (int c0 = 0; c0 < bsz; c0 += CH) {
                const int cn = min(CH, bsz - c0);
                // ---- gather + widen (iq_transform.cpp:17-20), targets -------
                for (int r = tid; r < cn; r += kT64) IDX[r] = perm[start + c0 + r];
                __syncthreads();
                for (int i = tid; i < cn * width; i += kT64) {
                    const int r = i / width, c = i % width, idx = IDX[r];
                    double v;
                    if (p.layout == NOMA_LAYOUT_WIDEN_COMPLEX) {
                        const double *x = p.design + ((size_t)d * (n / 2) + (idx >> 1)) * M * 2;
                        if (!(idx & 1)) v = c < M ? x[2 * c] : x[2 * (c - M) + 1];
                        else v = c < M ? x[2 * c + 1] : -x[2 * (c - M)];
                    } else {
                        v = p.design[((size_t)d * n + idx) * width + c];
                    }
                    ACT[aoff[0] + r * (width + 1) + c] = v;
                }
                for (int r = tid; r < cn; r += kT64) {
                    const int idx = IDX[r];
                    YB[r] = p.layout == NOMA_LAYOUT_WIDEN_COMPLEX
                                ? p.targets[(((size_t)d * (n / 2) + (idx >> 1)) * p.K + net % p.K) * 2 + (idx & 1)]
                                : p.targets[((size_t)d * p.K + net % p.K) * n + idx];
                }
                __syncthreads();
                // ---- forward (hybrid_nn.cpp:60-72) ---------------------------
                for (int l = 1; l <= N; ++l) {
                    const int in = g.dims[l - 1], out = g.dims[l];
                    const double *A = ACT + aoff[l - 1], *W = TH + woff[l], *B = TH + boff[l];
                    double *Z = ACT + aoff[l];
                    // register tiles of 2 rows (r, r + cn2) x 4 neurons per
                    // thread, rows across the lanes: the padded activation rows
                    // hit distinct banks, the weights broadcast; six loads per
                    // eight DFMA (each output still sums k in order)
                    const int cn2 = (cn + 1) >> 1, nq = (out + 3) >> 2;
                    for (int t = tid; t < cn2 * nq; t += kT64) {
                        const int rq = t % cn2, j0 = 4 * (t / cn2);
                        const int r1 = min(rq + cn2, cn - 1);
                        const double *a0 = A + rq * (in + 1), *a1 = A + r1 * (in + 1);
                        const double *w[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) w[u] = W + min(j0 + u, out - 1) * in;
                        double s0[4] = {0.0, 0.0, 0.0, 0.0}, s1[4] = {0.0, 0.0, 0.0, 0.0};
                        for (int k = 0; k < in; ++k) {
                            const double x0 = a0[k], x1 = a1[k];
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const double wk = w[u][k];
                                s0[u] += x0 * wk;
                                s1[u] += x1 * wk;
                            }
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int j = j0 + u;
                            if (j >= out) break;
                            const double z0 = s0[u] + B[j];
                            Z[rq * (out + 1) + j] = z0 > 0.0 ? z0 : 0.0;
                            if (rq + cn2 < cn) {
                                const double z1 = s1[u] + B[j];
                                Z[(rq + cn2) * (out + 1) + j] = z1 > 0.0 ? z1 : 0.0;
                            }
                        }
                    }
                    __syncthreads();
                }
                // ---- residual x w0 + a_N w - y, dy = 2 r / B (hybrid_nn.cpp:94-98)
                const int LN = g.dims[N];
                const double *AN = ACT + aoff[N];
                for (int r = tid; r < cn; r += kT64) {
                    double lin = 0.0, br = 0.0;
                    for (int c = 0; c < width; ++c) lin += ACT[aoff[0] + r * (width + 1) + c] * w0[c];
                    for (int c = 0; c < LN; ++c) br += AN[r * (LN + 1) + c] * TH[foff + c];
                    const double res = lin + br - YB[r];
                    sq += res * res;
                    YB[r] = (2.0 / (double)bsz) * res;  // dy
                }
                __syncthreads();
                // ---- final layer gradient, da = dy wf^T (hybrid_nn.cpp:99-102)
                for (int j = tid; j < LN; j += kT64) {
                    double s = 0.0;
                    for (int r = 0; r < cn; ++r) s += AN[r * (LN + 1) + j] * YB[r];
                    GR[foff + j] += s;
                }
                for (int i = tid; i < cn * LN; i += kT64) DA[i] = YB[i / LN] * TH[foff + i % LN];
                __syncthreads();
                // ---- hidden layers backward (hybrid_nn.cpp:105-112) ------------
                for (int l = N; l >= 1; --l) {
                    const int out = g.dims[l], in = g.dims[l - 1];
                    const double *A = ACT + aoff[l], *Ab = ACT + aoff[l - 1];
                    for (int i = tid; i < cn * out; i += kT64) DZ[i] = A[(i / out) * (out + 1) + i % out] > 0.0 ? DA[i] : 0.0;
                    __syncthreads();
                    {  // gW = dz^T below: tiles of 4 neurons x 2 columns (c, c + in2)
                        const int in2 = (in + 1) >> 1, nq = (out + 3) >> 2;
                        for (int t = tid; t < in2 * nq; t += kT64) {
                            const int cq = t % in2, j0 = 4 * (t / in2);
                            const int c1 = min(cq + in2, in - 1);
                            int jj[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) jj[u] = min(j0 + u, out - 1);
                            double s0[4] = {0.0, 0.0, 0.0, 0.0}, s1[4] = {0.0, 0.0, 0.0, 0.0};
                            for (int r = 0; r < cn; ++r) {
                                const double b0 = Ab[r * (in + 1) + cq], b1 = Ab[r * (in + 1) + c1];
#pragma unroll
                                for (int u = 0; u < 4; ++u) {
                                    const double zq = DZ[r * out + jj[u]];
                                    s0[u] += zq * b0;
                                    s1[u] += zq * b1;
                                }
                            }
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                if (j0 + u >= out) break;
                                GR[woff[l] + (j0 + u) * in + cq] += s0[u];
                                if (cq + in2 < in) GR[woff[l] + (j0 + u) * in + cq + in2] += s1[u];
                            }
                        }
                    }
                    for (int j = tid; j < out; j += kT64) {  // gb = colsum dz
                        double s = 0.0;
                        for (int r = 0; r < cn; ++r) s += DZ[r * out + j];
                        GR[boff[l] + j] += s;
                    }
                    if (l > 1) {  // da = dz W_l
                        // tiles of 4 rows x 2 columns (c, c + in2), columns across
                        // the lanes (contiguous weight reads), dz broadcast
                        const int in2 = (in + 1) >> 1, rq4 = (cn + 3) >> 2;
                        for (int t = tid; t < in2 * rq4; t += kT64) {
                            const int cq = t % in2, r0 = 4 * (t / in2);
                            const int c1 = min(cq + in2, in - 1);
                            int rr[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) rr[u] = min(r0 + u, cn - 1);
                            double s0[4] = {0.0, 0.0, 0.0, 0.0}, s1[4] = {0.0, 0.0, 0.0, 0.0};
                            for (int j = 0; j < out; ++j) {
                                const double t0 = TH[woff[l] + j * in + cq], t1 = TH[woff[l] + j * in + c1];
#pragma unroll
                                for (int u = 0; u < 4; ++u) {
                                    const double zq = DZ[rr[u] * out + j];
                                    s0[u] += zq * t0;
                                    s1[u] += zq * t1;
                                }
                            }
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                if (r0 + u >= cn) break;
                                DA[(r0 + u) * in + cq] = s0[u];
                                if (cq + in2 < in) DA[(r0 + u) * in + cq + in2] = s1[u];
                            }
                        }
                    }
                    __syncthreads();
                }
            }
            // ---- loss of the step and Adam (hybrid_nn.cpp:118-144) ------------
            RED[tid] = sq;
            __syncthreads();
            if (tid == 0) {
                double s = 0.0;
                for (int i = 0; i < kT64; ++i) s += RED[i];
                const double loss = s / (double)bsz;
                loss_sum += loss * (double)bsz;
            }
            ++step;
            const double corr1 = 1.0 - pow(p.b1, (double)step);
            const double corr2 = 1.0 - pow(p.b2, (double)step);
            // moments live in global memory (L2): four parameters per thread
            // at a time so that their eight loads are in flight together
            for (int i0 = tid; i0 < p.ptrain; i0 += 4 * kT64) {
                double pm1[4], pm2[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = min(i0 + u * kT64, p.ptrain - 1);
                    pm1[u] = m1[i];
                    pm2[u] = m2[i];
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = i0 + u * kT64;
                    if (i >= p.ptrain) break;
                    const double gi = GR[i];
                    const double a = p.b1 * pm1[u] + (1.0 - p.b1) * gi;
                    const double b = p.b2 * pm2[u] + (1.0 - p.b2) * (gi * gi);
                    m1[i] = a;
                    m2[i] = b;
                    TH[i] -= p.lr * (a / corr1) / (sqrt(b / corr2) + p.eps);
                }
            }
            __syncthreads();
        }
        if (tid == 0 && p.trace) p.trace[(size_t)net * p.epochs + e] = loss_sum / (double)n;
    }
    for (int i = tid; i < p.ptrain; i += kT64) gtheta[i] = TH[i];
}

int train_f64_launch(TrainF64Params &p, cudaStream_t st) {
    const NetGeom &g = p.g;
    if (p.batch < 1) return NOMA_ERR_CONFIG;
    p.ptrain = trainable_count(g);
    // one hidden layer of 64 on a 32 / 64-wide input: register-tiled DFMA kernel
    if (train_w8d_fits(p)) {
        p.mode = 301;
        return train_w8d_launch(p, st);
    }
    p.mode = 300;
    int maxw = 0;
    for (int l = 0; l < g.nd; ++l) maxw = g.dims[l] > maxw ? g.dims[l] : maxw;
    p.maxw = maxw;
    p.ptrain = trainable_count(g);
    for (int ch = 128; ch >= 8; ch /= 2) {
        int act = 0;
        for (int l = 0; l < g.nd; ++l) act += ch * (g.dims[l] + 1);
        const size_t smem = (size_t)(2 * p.ptrain + act + 2 * ch * maxw + ch + kT64) * sizeof(double) +
                            ch * sizeof(int);
        if (smem <= 227 * 1024) {
            p.chunk = ch;
            p.act_total = act;
            cudaFuncSetAttribute(train_f64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            train_f64_kernel<<<p.n_nets, kT64, smem, st>>>(p);
            return cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;
        }
    }
    return NOMA_ERR_UNSUPPORTED;
}

}  // namespace noma_dev
