// Bit-exact RNG consumers on sm_100a: per-epoch Fisher-Yates shuffles
// (hybrid_nn.cpp:148-154, :176), He-normal initialisation (hybrid_nn.cpp:34-55)
// and the synthetic uplink generator (channel_sim.cpp:30-117).
//
// Every reference stream is sequential (xoshiro256++), so the unit of
// parallelism is the stream: one thread per (net, epoch) shuffle, one thread
// per net initialisation, one thread per slot for the synthesiser's draws.
// The data-parallel parts (superposition, distortion, noise scaling) run one
// thread per receive sample.
#include <math.h>

#include "kernels.cuh"

namespace noma_dev {

// ---------------------------------------------------------------- shuffle
// perm[net][epoch][n] (u16).  Each thread owns one (net, epoch) and keeps its
// index array in shared memory while applying the 1..n-1 swaps.
__global__ void perm_kernel(int n_nets, int epochs, int n, const uint64_t *shuffle_seeds,
                            uint16_t *perm) {
    extern __shared__ uint16_t sidx[];
    const int job = blockIdx.x * blockDim.x + threadIdx.x;
    if (job >= n_nets * epochs) return;
    const int net = job / epochs, epoch = job % epochs;
    uint16_t *idx = sidx + (size_t)threadIdx.x * n;
    for (int i = 0; i < n; ++i) idx[i] = (uint16_t)i;
    Xoshiro r(substream_seed(shuffle_seeds[net], (uint64_t)epoch));
    for (int i = n - 1; i > 0; --i) {
        const int j = (int)r.below((uint64_t)i + 1);
        const uint16_t t = idx[i];
        idx[i] = idx[j];
        idx[j] = t;
    }
    uint16_t *out = perm + (size_t)job * n;
    for (int i = 0; i < n; ++i) out[i] = idx[i];
}

int perm_launch(int n_nets, int epochs, int n, const uint64_t *seeds, uint16_t *perm,
                cudaStream_t st) {
    if (n > 65535) return NOMA_ERR_UNSUPPORTED;
    const int jobs = n_nets * epochs;
    if (jobs == 0) return NOMA_OK;
    int tpb = (int)((160 * 1024) / (2 * (size_t)n));
    tpb = tpb > 64 ? 64 : tpb;
    if (tpb < 1) return NOMA_ERR_UNSUPPORTED;
    const size_t smem = (size_t)tpb * n * sizeof(uint16_t);
    cudaFuncSetAttribute(perm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    perm_kernel<<<(jobs + tpb - 1) / tpb, tpb, smem, st>>>(n_nets, epochs, n, seeds, perm);
    return cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;
}

// ------------------------------------------------------------------- init
// He-normal initialisation (hybrid_nn.cpp:43-52), one CTA per net.  The
// reference stream is sequential, so one producer thread runs xoshiro256++
// ahead into a double-buffered shared-memory ring of raw u64 pairs while the
// other threads turn the previous chunk into Box-Muller draws (the FP64
// log/sqrt/cos dominate the per-draw cost) and scatter them into the plan
// (FP32, FusedPlan layout) and/or the flat FP64 parameter vector.
// Seeds come from `seeds` (Rng(seed)) or, when `states` is non-null, from
// caller xoshiro states that are advanced in place (init_params(..., Rng&)).
constexpr int kInitThreads = 128;
constexpr int kInitChunk = 1024;  // gaussians per ring slot

__global__ void __launch_bounds__(kInitThreads) init_block_kernel(
    NetGeom g, const uint64_t *seeds, uint64_t *states, const double *w0, float *plans,
    double *theta, int ptrain) {
    __shared__ uint64_t ring[2][2 * kInitChunk];
    const int net = blockIdx.x, tid = threadIdx.x;
    float *pl = plans ? plans + (size_t)net * g.plan_total : nullptr;
    double *th = theta ? theta + (size_t)net * ptrain : nullptr;
    // zero outputs, w0 slot, biases / final (theta)
    if (pl) {
        for (int i = tid; i < g.plan_total; i += kInitThreads) pl[i] = 0.0f;
    }
    if (th) {
        for (int i = tid; i < ptrain; i += kInitThreads) th[i] = 0.0;
    }
    __syncthreads();
    if (pl && w0)
        for (int c = tid; c < g.dims[0]; c += kInitThreads) pl[c] = (float)w0[(size_t)net * g.dims[0] + c];
    // gaussian count and per-layer starts (reference draw order)
    int start[NOMA_MAX_DIMS + 1];
    int total = 0;
    for (int l = 1; l < g.nd; ++l) {
        start[l] = total;
        total += g.dims[l] * g.dims[l - 1];
    }
    start[g.nd] = total;
    Xoshiro r = states ? Xoshiro(states[net * 4], states[net * 4 + 1], states[net * 4 + 2], states[net * 4 + 3])
                       : Xoshiro(seeds[net]);
    const int chunks = (total + kInitChunk - 1) / kInitChunk;
    auto produce = [&](int c) {
        const int n = min(kInitChunk, total - c * kInitChunk);
        uint64_t *b = ring[c & 1];
        for (int i = 0; i < 2 * n; ++i) b[i] = r.next();
    };
    if (tid == 0 && chunks > 0) produce(0);
    __syncthreads();
    for (int c = 0; c < chunks; ++c) {
        if (tid == 0) {
            if (c + 1 < chunks) produce(c + 1);
        } else {
            const int n = min(kInitChunk, total - c * kInitChunk);
            const uint64_t *b = ring[c & 1];
            for (int i = tid - 1; i < n; i += kInitThreads - 1) {
                const int w = c * kInitChunk + i;
                int l = 1;
                while (w >= start[l + 1]) ++l;
                const int fan_in = g.dims[l - 1];
                const int off = w - start[l], row = off / fan_in, col = off % fan_in;
                // Box-Muller cosine half (rng.hpp:58-62) on the recorded pair
                const double u1 = 1.0 - static_cast<double>(b[2 * i] >> 11) * 0x1.0p-53;
                const double u2 = static_cast<double>(b[2 * i + 1] >> 11) * 0x1.0p-53;
                const double ang = __dmul_rn(2.0 * 3.141592653589793238462643383279502884, u2);
                const double gauss = __dmul_rn(sqrt(__dmul_rn(-2.0, log(u1))), cos(ang));
                const double v = gauss * sqrt(2.0 / fan_in);
                if (pl) pl[g.plan_w[l] + row * g.plan_pad[l - 1] + col] = (float)v;
                if (th) {
                    int t = 0;  // flat offset: W_1, b_1, ..., W_l block
                    for (int q = 1; q < l; ++q) t += g.dims[q] * g.dims[q - 1] + g.dims[q];
                    th[t + off] = v;
                }
            }
        }
        __syncthreads();
    }
    if (states && tid == 0) {
        states[net * 4] = r.s0;
        states[net * 4 + 1] = r.s1;
        states[net * 4 + 2] = r.s2;
        states[net * 4 + 3] = r.s3;
    }
}

int init_state_launch(const NetGeom &g, int n_nets, uint64_t *states, const double *w0,
                      float *plans, double *theta, int ptrain, cudaStream_t st) {
    if (n_nets == 0) return NOMA_OK;
    init_block_kernel<<<n_nets, kInitThreads, 0, st>>>(g, nullptr, states, w0, plans, theta, ptrain);
    return cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;
}

int init_launch(const NetGeom &g, int n_nets, const uint64_t *seeds, const double *w0,
                float *plans, cudaStream_t st) {
    if (n_nets == 0) return NOMA_OK;
    init_block_kernel<<<n_nets, kInitThreads, 0, st>>>(g, seeds, nullptr, w0, plans, nullptr, 0);
    return cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;
}

// Copies FP64 w0 [net][d0] into the plans' w0 slots.
__global__ void set_w0_kernel(int n_nets, int d0, int plan_total, const double *w0,
                              float *plans) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_nets * d0) return;
    const int net = i / d0, c = i % d0;
    plans[(size_t)net * plan_total + c] = (float)w0[i];
}

int set_w0_launch(int n_nets, int d0, int plan_total, const double *w0, float *plans,
                  cudaStream_t st) {
    const int n = n_nets * d0;
    if (n == 0) return NOMA_OK;
    set_w0_kernel<<<(n + 255) / 256, 256, 0, st>>>(n_nets, d0, plan_total, w0, plans);
    return cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;
}

// -------------------------------------------------------------- synthesis
// One thread per slot: the three sequential streams of SeedBundle.
__global__ void synth_draw_kernel(SynthParams p) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= p.S) return;
    const uint64_t master = p.bundles ? 0 : p.seeds[s];
    Xoshiro sym(p.bundles ? p.seeds[3 * s] : substream_seed(master, 1)),
        chan(p.bundles ? p.seeds[3 * s + 1] : substream_seed(master, 2)),
        noise(p.bundles ? p.seeds[3 * s + 2] : substream_seed(master, 3));
    const double hs = 1.0 / sqrt(2.0);
    double *h = p.channel + (size_t)s * p.M * p.K * 2;
    for (int k = 0; k < p.K; ++k)  // gen_channel: k then m; g++ draws imag first
        for (int m = 0; m < p.M; ++m) {
            const double im = __dmul_rn(chan.gaussian(), hs);
            const double re = __dmul_rn(chan.gaussian(), hs);
            h[((size_t)m * p.K + k) * 2] = re;
            h[((size_t)m * p.K + k) * 2 + 1] = im;
        }
    const int T = p.NT + p.ND;
    uint8_t *codes = p.codes_all + (size_t)s * T * p.K;
    for (int t = 0; t < T; ++t)
        for (int k = 0; k < p.K; ++k) codes[(size_t)t * p.K + k] = (uint8_t)sym.below(4);
    double np = 0.0;
    if (p.noisy) {
        double sig = 0.0;
        for (int k = 0; k < p.K; ++k) {
            double nrm = 0.0;
            for (int m = 0; m < p.M; ++m) {
                const double re = h[((size_t)m * p.K + k) * 2], im = h[((size_t)m * p.K + k) * 2 + 1];
                nrm = __dadd_rn(nrm, __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im)));
            }
            sig = __dadd_rn(sig, __dmul_rn(p.powers[k], nrm));
        }
        np = sig / __dmul_rn((double)p.M, p.snr_lin);
        double *nz = p.noise + (size_t)s * T * p.M * 2;
        for (int t = 0; t < T; ++t)
            for (int m = 0; m < p.M; ++m) {
                const double im = noise.gaussian();
                const double re = noise.gaussian();
                nz[((size_t)t * p.M + m) * 2] = re;
                nz[((size_t)t * p.M + m) * 2 + 1] = im;
            }
    }
    if (p.noise_power) p.noise_power[s] = np;
}

// One thread per (slot, t, m): superposition, cubic distortion, noise.
__global__ void synth_mix_kernel(SynthParams p, const double *noise_power) {
    const int T = p.NT + p.ND;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)p.S * T * p.M) return;
    const int m = (int)(i % p.M);
    const int t = (int)((i / p.M) % T);
    const int s = (int)(i / ((size_t)p.M * T));
    const double a = 1.0 / sqrt(2.0);
    const double *h = p.channel + (size_t)s * p.M * p.K * 2;
    const uint8_t *codes = p.codes_all + ((size_t)s * T + t) * p.K;
    double re = 0.0, im = 0.0;
    for (int k = 0; k < p.K; ++k) {
        const uint8_t b = codes[k];
        const double br = (b & 1) ? -a : a, bi = (b & 2) ? -a : a;
        const double sp = sqrt(p.powers[k]);
        const double cr = __dmul_rn(h[((size_t)m * p.K + k) * 2], sp);
        const double ci = __dmul_rn(h[((size_t)m * p.K + k) * 2 + 1], sp);
        re = __dadd_rn(re, __dsub_rn(__dmul_rn(br, cr), __dmul_rn(bi, ci)));
        im = __dadd_rn(im, __dadd_rn(__dmul_rn(br, ci), __dmul_rn(bi, cr)));
    }
    if (p.gain > 0.0) {
        const double nrm = __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im));
        re = __dadd_rn(re, __dmul_rn(__dmul_rn(p.gain, re), nrm));
        im = __dadd_rn(im, __dmul_rn(__dmul_rn(p.gain, im), nrm));
    }
    if (p.noisy) {
        const double sd = sqrt(noise_power[s] / 2.0);
        const double *nz = p.noise + (((size_t)s * T + t) * p.M + m) * 2;
        re = __dadd_rn(re, __dmul_rn(nz[0], sd));
        im = __dadd_rn(im, __dmul_rn(nz[1], sd));
    }
    if (t < p.NT) {
        if (p.pilot_rx) {
            double *o = p.pilot_rx + (((size_t)s * p.NT + t) * p.M + m) * 2;
            o[0] = re;
            o[1] = im;
        }
        if (p.pilot_sym && m < p.K) {  // piggy-back: symbols of this row
            const double br = (codes[m] & 1) ? -a : a, bi = (codes[m] & 2) ? -a : a;
            double *o = p.pilot_sym + (((size_t)s * p.NT + t) * p.K + m) * 2;
            o[0] = br;
            o[1] = bi;
        }
    } else {
        const int td = t - p.NT;
        if (p.data_rx) {
            float *o = p.data_rx + (((size_t)s * p.ND + td) * p.M + m) * 2;
            o[0] = (float)re;
            o[1] = (float)im;
        }
        if (p.data_codes && m < p.K) p.data_codes[((size_t)s * p.ND + td) * p.K + m] = codes[m];
    }
}

// pilot symbols / data codes for users k >= M (the mix kernel covers k < M)
__global__ void synth_codes_tail_kernel(SynthParams p) {
    const int T = p.NT + p.ND;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int extra = p.K - p.M;
    if (extra <= 0 || i >= (size_t)p.S * T * extra) return;
    const int k = p.M + (int)(i % extra);
    const int t = (int)((i / extra) % T);
    const int s = (int)(i / ((size_t)extra * T));
    const double a = 1.0 / sqrt(2.0);
    const uint8_t c = p.codes_all[((size_t)s * T + t) * p.K + k];
    if (t < p.NT) {
        if (p.pilot_sym) {
            double *o = p.pilot_sym + (((size_t)s * p.NT + t) * p.K + k) * 2;
            o[0] = (c & 1) ? -a : a;
            o[1] = (c & 2) ? -a : a;
        }
    } else if (p.data_codes) {
        p.data_codes[((size_t)s * p.ND + (t - p.NT)) * p.K + k] = c;
    }
}

int synth_launch(SynthParams p, double *noise_power_scratch, cudaStream_t st) {
    const int T = p.NT + p.ND;
    synth_draw_kernel<<<(p.S + 63) / 64, 64, 0, st>>>(p);
    if (cudaGetLastError() != cudaSuccess) return NOMA_ERR_CUDA;
    const size_t n = (size_t)p.S * T * p.M;
    synth_mix_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(p, noise_power_scratch);
    if (cudaGetLastError() != cudaSuccess) return NOMA_ERR_CUDA;
    if (p.K > p.M) {
        const size_t n2 = (size_t)p.S * T * (p.K - p.M);
        synth_codes_tail_kernel<<<(unsigned)((n2 + 255) / 256), 256, 0, st>>>(p);
        if (cudaGetLastError() != cudaSuccess) return NOMA_ERR_CUDA;
    }
    return NOMA_OK;
}

}  // namespace noma_dev
