// Shared device/host helpers for the sm_100a NOMA detector kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "noma_cuda.h"

namespace noma_dev {

constexpr int kThreads = 256;     // CTA size of the train / detect / LLS kernels
constexpr int kBatchRows = 128;   // minibatch tile (NOMA_MAX_BATCH)
// Cycle probes (NOMA_PHASE_CLOCKS, NOMA_PHASE_TRACE, NOMA_LLS_CLOCKS,
// NOMA_DETECT_CLK) exist only in a build with -DNOMA_PROBES
// (NOMA_BUILD_TRACE=1 python -m paper_2206_05998_b200.build): predicated off
// they still cost the latency kernel ~8 % of a C1 slot (same-box A/B).
#ifdef NOMA_PROBES
#define NOMA_PROBE_ON(cond) (cond)
#else
#define NOMA_PROBE_ON(cond) false
#endif
constexpr int kSR = kBatchRows + 4;  // feature-major row stride: 132 == 4 (mod 32)
constexpr int kFeatPad = 32;      // every feature dim padded to 32 on chip

__host__ __device__ inline int pad_to(int w, int m) { return ((w + m - 1) / m) * m; }

#ifdef __CUDACC__
// Adam parameter step lr_t m / (sqrt(v / (1 - b2^t)) + eps) (hybrid_nn.cpp:133-139)
// with the single-instruction approximate square root (MUFU.SQRT, ~1 ulp):
// the IEEE sqrtf sequence cost ~8 instructions per parameter update, a
// visible share of the training kernels; the difference is far below the
// FP32 training's own rounding against the FP64 reference
__device__ __forceinline__ float adam_step(float lr_m1, float m2_ic2, float eps) {
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(m2_ic2));
    return __fdividef(lr_m1, r + eps);
}
#endif

// ------------------------------------------------------------------ RNG
// rng.hpp:10-62, bit-exact: splitmix64, substream_seed, xoshiro256++,
// 53-bit uniform, multiply-shift below(), Box-Muller cosine half.
__host__ __device__ inline uint64_t splitmix64(uint64_t &state) {
    uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__host__ __device__ inline uint64_t substream_seed(uint64_t master, uint64_t tag) {
    uint64_t s = master;
    uint64_t a = splitmix64(s);
    s = a ^ (tag * 0xD1B54A32D192ED03ULL + 0x8BB84B93962EACC9ULL);
    return splitmix64(s);
}

struct Xoshiro {
    uint64_t s0, s1, s2, s3;
    __host__ __device__ Xoshiro(uint64_t a, uint64_t b, uint64_t c, uint64_t d)
        : s0(a), s1(b), s2(c), s3(d) {}
    __host__ __device__ explicit Xoshiro(uint64_t seed) {
        uint64_t sm = seed;
        s0 = splitmix64(sm);
        s1 = splitmix64(sm);
        s2 = splitmix64(sm);
        s3 = splitmix64(sm);
    }
    __host__ __device__ static inline uint64_t rotl(uint64_t x, int k) {
        return (x << k) | (x >> (64 - k));
    }
    __host__ __device__ inline uint64_t next() {
        const uint64_t result = rotl(s0 + s3, 23) + s0;
        const uint64_t t = s1 << 17;
        s2 ^= s0;
        s3 ^= s1;
        s1 ^= s2;
        s0 ^= s3;
        s2 ^= t;
        s3 = rotl(s3, 45);
        return result;
    }
    __host__ __device__ inline double uniform() {
        return static_cast<double>(next() >> 11) * 0x1.0p-53;
    }
    __device__ inline uint64_t below(uint64_t bound) { return __umul64hi(next(), bound); }
    __device__ inline double gaussian() {
        const double u1 = 1.0 - uniform();
        const double u2 = uniform();
        // 2*pi*u2 evaluated as (2*pi)*u2 like the reference; no FMA contraction.
        const double ang = __dmul_rn(2.0 * 3.141592653589793238462643383279502884, u2);
        return __dmul_rn(sqrt(__dmul_rn(-2.0, log(u1))), cos(ang));
    }
};

// ------------------------------------------------------ network geometry
// FusedPlan layout (fused_inference.cpp:19-42) and the on-chip layout of the
// same parameters: every feature dim padded to kFeatPad, weight rows strided
// SW_l = FP_{l-1} + 4 (== 4 mod 32) so float4 row reads are conflict-free.
struct NetGeom {
    int nd;                        // dims count (input + hidden)
    int dims[NOMA_MAX_DIMS];
    int fp[NOMA_MAX_DIMS];         // on-chip feature pad (multiple of 32)
    int sw[NOMA_MAX_DIMS];         // on-chip W_l row stride, l >= 1
    int pw[NOMA_MAX_DIMS], pb[NOMA_MAX_DIMS], pf, ptotal;  // on-chip param block
    int plan_w0, plan_w[NOMA_MAX_DIMS], plan_b[NOMA_MAX_DIMS], plan_f, plan_total;
    int plan_pad[NOMA_MAX_DIMS];   // pad8 widths of the plan
    int maxfp;                     // max fp over hidden layers and input
};

inline bool make_geom(const noma_net_desc *d, NetGeom *g) {
    if (!d || d->ndims < 1 || d->ndims > NOMA_MAX_DIMS) return false;
    g->nd = d->ndims;
    g->maxfp = 0;
    for (int l = 0; l < d->ndims; ++l) {
        if (d->dims[l] < 1) return false;
        g->dims[l] = d->dims[l];
        g->fp[l] = pad_to(d->dims[l], kFeatPad);
        g->plan_pad[l] = pad_to(d->dims[l], 8);
        g->maxfp = g->fp[l] > g->maxfp ? g->fp[l] : g->maxfp;
    }
    int off = 0;
    g->sw[0] = 0;
    g->pw[0] = g->pb[0] = 0;
    for (int l = 1; l < g->nd; ++l) {
        g->sw[l] = g->fp[l - 1] + 4;
        g->pw[l] = off;
        off += g->fp[l] * g->sw[l];
        g->pb[l] = off;
        off += g->fp[l];
    }
    g->pf = off;
    off += g->fp[g->nd - 1];
    g->ptotal = off;
    // plan
    int po = g->plan_pad[0];
    g->plan_w0 = 0;
    g->plan_w[0] = g->plan_b[0] = 0;
    for (int l = 1; l < g->nd; ++l) {
        g->plan_w[l] = po;
        po += g->dims[l] * g->plan_pad[l - 1];
        g->plan_b[l] = po;
        po += g->plan_pad[l];
    }
    g->plan_f = po;
    po += g->plan_pad[g->nd - 1];
    g->plan_total = po;
    return true;
}

inline int trainable_count(const NetGeom &g) {
    int n = g.dims[g.nd - 1];
    for (int l = 1; l < g.nd; ++l) n += g.dims[l] * g.dims[l - 1] + g.dims[l];
    return n;
}

}  // namespace noma_dev
