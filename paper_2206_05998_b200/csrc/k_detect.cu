// Data-phase detection on sm_100a: replaces hybrid_nn::detect
// (hybrid_nn.cpp:197-199) / fused::fused_forward_f32 (fused_inference.cpp:
// 222-231) with hard_decision_qpsk and bit_error_rate (eval.cpp:38-65) fused
// into the epilogue.
//
// Grid (ctas_per_net, n_nets).  Each CTA keeps one user's network resident
// in shared memory and streams 64-symbol tiles (128 widened rows) of its
// slot's data: coalesced complex loads, IQ widening while transposing into
// the feature-major tile, the same FP32 register-tile forward as training,
// then the linear branch, the QPSK sign decision and a warp-reduced bit-error
// count (one atomic per warp per tile).
#include <cstdlib>

#include "kernels.cuh"
#include "tiles.cuh"

namespace noma_dev {

__global__ void __launch_bounds__(kThreads) detect_kernel(DetectParams p) {
    extern __shared__ __align__(16) float sm[];
    const int net = blockIdx.y, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (p.status && p.status[net] != NOMA_OK) {
        if (blockIdx.x == 0 && tid == 0 && p.errors) p.errors[net] = 0xFFFFFFFFu;
        if (blockIdx.x == 0 && tid == 0 && p.sym_errors) p.sym_errors[net] = 0xFFFFFFFFu;
        return;
    }
    const NetGeom &g = p.g;
    const int N = g.nd - 1, d = net / p.K, k = net % p.K;
    float *XT = sm + p.off_x, *PS = sm + p.off_ps, *W0 = sm + p.off_w0, *Y = sm + p.off_y;
    float *YP = sm + p.off_yp;
    float *buf[2] = {sm + p.off_a0, sm + p.off_a1};

    for (int i = tid; i < p.off_end; i += kThreads) sm[i] = 0.0f;
    __syncthreads();
    const float *pl = p.plans + (size_t)net * g.plan_total;
    for (int c = tid; c < g.dims[0]; c += kThreads) W0[c] = pl[c];
    for (int l = 1; l <= N; ++l) {
        const int rowsl = g.dims[l], cols = g.dims[l - 1];
        for (int i = tid; i < rowsl * cols; i += kThreads) {
            const int j = i / cols, c = i % cols;
            PS[g.pw[l] + j * g.sw[l] + c] = pl[g.plan_w[l] + j * g.plan_pad[l - 1] + c];
        }
        for (int j = tid; j < rowsl; j += kThreads) PS[g.pb[l] + j] = pl[g.plan_b[l] + j];
    }
    for (int j = tid; j < g.dims[N]; j += kThreads) PS[g.pf + j] = pl[g.plan_f + j];
    __syncthreads();

    const bool widen = p.layout == NOMA_LAYOUT_WIDEN_COMPLEX;
    const int M = p.width / 2;
    const int rows_per_tile = widen ? kBatchRows / 2 : kBatchRows;  // symbols or rows
    uint32_t my_err = 0, my_ser = 0;
    for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
        const int t0 = tile * rows_per_tile;
        const int tn = min(rows_per_tile, p.rows - t0);
        // ---- gather + widen ------------------------------------------------
        if (widen) {
            const float2 *src = reinterpret_cast<const float2 *>(p.data) + ((size_t)d * p.stride + t0) * M;
            for (int i = tid; i < rows_per_tile * M; i += kThreads) {
                const int tl = i / M, m = i % M;
                float2 v = make_float2(0.f, 0.f);
                if (tl < tn) v = src[i];
                XT[m * kSR + 2 * tl] = v.x;
                XT[(M + m) * kSR + 2 * tl] = v.y;
                XT[m * kSR + 2 * tl + 1] = v.y;
                XT[(M + m) * kSR + 2 * tl + 1] = -v.x;
            }
        } else {
            const float *src = p.data + ((size_t)d * p.stride + t0) * p.width;
            for (int i = tid; i < rows_per_tile * p.width; i += kThreads) {
                const int r = i / p.width, c = i % p.width;
                XT[c * kSR + r] = r < tn ? src[i] : 0.0f;
            }
        }
        __syncthreads();
        // ---- hidden layers ---------------------------------------------------
        const float *in = XT;
        for (int l = 1; l <= N; ++l) {
            float *out = buf[(l - 1) & 1];
            tile_forward<kThreads / 32>(PS + g.pw[l], g.sw[l], PS + g.pb[l], in, out, g.fp[l],
                                        g.fp[l - 1], warp, lane, l == N ? PS + g.pf : nullptr,
                                        l == N ? YP : nullptr);
            __syncthreads();
            in = out;
        }
        // ---- linear branch + final layer (fused_inference.cpp:84-91, :118-125)
        if (tid < kBatchRows) {
            float lin = 0.0f;
            for (int c = 0; c < g.fp[0]; ++c) lin = fmaf(W0[c], XT[c * kSR + tid], lin);
            float br = 0.0f;
            if (N) {
                for (int b = 0; b < (g.fp[N] >> 5); ++b) br += YP[b * kBatchRows + tid];
            } else {
                const float *wf = PS + g.pf;
                for (int j = 0; j < g.fp[N]; ++j) br = fmaf(wf[j], in[j * kSR + tid], br);
            }
            Y[tid] = lin + br;
        }
        __syncthreads();
        // ---- epilogue: soft output, hard decision, bit errors ---------------
        if (widen) {
            if (tid < kBatchRows / 2) {
                const int t = t0 + tid;
                uint32_t e = 0;
                if (tid < tn) {
                    const float re = Y[2 * tid], im = Y[2 * tid + 1];
                    const uint8_t code = (uint8_t)((re < 0.0f ? 1 : 0) | (im < 0.0f ? 2 : 0));
                    if (p.soft)
                        reinterpret_cast<float2 *>(p.soft)[(size_t)net * p.stride + t] = make_float2(re, im);
                    if (p.codes) p.codes[(size_t)net * p.stride + t] = code;
                    if (p.truth) e = __popc((code ^ p.truth[((size_t)d * p.stride + t) * p.K + k]) & 3u);
                }
                my_err += e;
                my_ser += e ? 1u : 0u;
            }
        } else if (tid < tn && p.soft) {
            p.soft[(size_t)net * p.stride + t0 + tid] = Y[tid];
        }
        __syncthreads();
    }
    if ((p.errors || p.sym_errors) && p.truth && warp < 2) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            my_err += __shfl_xor_sync(0xffffffffu, my_err, o);
            my_ser += __shfl_xor_sync(0xffffffffu, my_ser, o);
        }
        if (lane == 0 && my_err && p.errors) atomicAdd(p.errors + net, my_err);
        if (lane == 0 && my_ser && p.sym_errors) atomicAdd(p.sym_errors + net, my_ser);
    }
}

int detect_launch(DetectParams &p, cudaStream_t st) {
    const NetGeom &g = p.g;
    // tensor-core path (k_detect_tc.cu) for the shapes it covers, unless
    // NOMA_DETECT_TC=0 (A/B and parity runs of the FFMA kernel)
    const char *tc_env = std::getenv("NOMA_DETECT_TC");
    if (!(tc_env && tc_env[0] == '0')) {
        const int r = detect_tc_launch(p, st);
        if (r != NOMA_ERR_UNSUPPORTED) {
            p.mode = 2;
            return r;
        }
    }
    p.mode = 1;
    for (int l = 0; l < g.nd; ++l)
        if (g.dims[l] > NOMA_MAX_WIDTH) return NOMA_ERR_UNSUPPORTED;
    int maxh = 32;
    for (int l = 1; l < g.nd; ++l) maxh = g.fp[l] > maxh ? g.fp[l] : maxh;
    int off = 0;
    p.off_x = off;
    off += g.fp[0] * kSR;
    p.off_a0 = off;
    off += maxh * kSR;
    p.off_a1 = off;
    off += maxh * kSR;
    p.off_ps = off;
    off += pad_to(g.ptotal, 4);
    p.off_w0 = off;
    off += g.fp[0];
    p.off_y = off;
    off += kBatchRows;
    p.off_yp = off;
    off += (g.fp[g.nd - 1] / 32) * kBatchRows;
    p.off_end = off;
    const size_t smem = (size_t)off * sizeof(float);
    if (smem > 227 * 1024) return NOMA_ERR_UNSUPPORTED;
    const int rows_per_tile = p.layout == NOMA_LAYOUT_WIDEN_COMPLEX ? kBatchRows / 2 : kBatchRows;
    p.tiles = (p.rows + rows_per_tile - 1) / rows_per_tile;
    if (p.stride == 0) p.stride = p.rows;
    if (p.tiles == 0 || p.n_nets == 0) return NOMA_OK;
    // one wave of resident CTAs split evenly over the nets (rounded down: a
    // partial second wave would double the time of a few-net launch)
    cudaFuncSetAttribute(detect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int sms = 148, dev = 0, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, detect_kernel, kThreads, smem) != cudaSuccess ||
        per_sm < 1) {
        cudaGetLastError();
        per_sm = 1;
    }
    int ctas = sms * per_sm / p.n_nets;
    ctas = ctas < 1 ? 1 : ctas;
    ctas = ctas > p.tiles ? p.tiles : ctas;
    detect_kernel<<<dim3(ctas, p.n_nets), kThreads, smem, st>>>(p);
    return cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;
}

}  // namespace noma_dev
