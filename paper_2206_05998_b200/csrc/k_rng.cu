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

#include <mutex>
#include <vector>

#include "kernels.cuh"

namespace noma_dev {

// ------------------------------------------------------------ jump-ahead
// xoshiro256's state update (rng.hpp:35-45, without the ++ output scrambler)
// is linear over GF(2): s' = T s with T a 256x256 bit matrix.  With
// J = T^kJumpDraws precomputed, the state before draw c*kJumpDraws is J^c s0,
// so independent threads can generate consecutive blocks of one reference
// stream -- bit-identical draws, in parallel.  Tables (rows = 4 x u64 per
// output bit): lo[b] = J^b (b < kJumpLo), hi[a] = J^(kJumpLo a) (a < kJumpHi),
// built once per device on the host.
constexpr int kJumpDraws = 128;
constexpr int kJumpLo = 64, kJumpHi = 64;  // up to 4096 blocks = 524288 draws

namespace {
struct Gf2 {
    uint64_t r[256][4];
};
void gf2_mul(const Gf2 &a, const Gf2 &b, Gf2 &out) {  // out = a . b (row form)
    for (int i = 0; i < 256; ++i) {
        uint64_t acc[4] = {0, 0, 0, 0};
        for (int k = 0; k < 256; ++k)
            if ((a.r[i][k >> 6] >> (k & 63)) & 1)
                for (int w = 0; w < 4; ++w) acc[w] ^= b.r[k][w];
        for (int w = 0; w < 4; ++w) out.r[i][w] = acc[w];
    }
}
void gf2_step_matrix(Gf2 &t) {  // T: column j = one xoshiro step of e_j
    for (int i = 0; i < 256; ++i)
        for (int w = 0; w < 4; ++w) t.r[i][w] = 0;
    for (int j = 0; j < 256; ++j) {
        uint64_t s[4] = {0, 0, 0, 0};
        s[j >> 6] = 1ull << (j & 63);
        Xoshiro x(s[0], s[1], s[2], s[3]);
        x.next();
        const uint64_t o[4] = {x.s0, x.s1, x.s2, x.s3};
        for (int i = 0; i < 256; ++i)
            if ((o[i >> 6] >> (i & 63)) & 1) t.r[i][j >> 6] |= 1ull << (j & 63);
    }
}
std::mutex g_jump_mu;
const uint64_t *g_jump[64] = {};  // per device: lo tables then hi tables
}  // namespace

// Device table [kJumpLo + kJumpHi][256][4] for the current device (cached).
const uint64_t *jump_table() {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_jump_mu);
    if (dev < 0 || dev >= 64) return nullptr;
    if (g_jump[dev]) return g_jump[dev];
    std::vector<Gf2> tab(kJumpLo + kJumpHi);
    Gf2 t, j, tmp;
    gf2_step_matrix(t);
    j = t;  // J = T^128 by squaring (128 = 2^7)
    for (int k = 0; k < 7; ++k) {
        gf2_mul(j, j, tmp);
        j = tmp;
    }
    for (int i = 0; i < 256; ++i)
        for (int w = 0; w < 4; ++w) tab[0].r[i][w] = (w == (i >> 6)) ? 1ull << (i & 63) : 0;
    for (int b = 1; b < kJumpLo; ++b) gf2_mul(tab[b - 1], j, tab[b]);
    Gf2 big;
    gf2_mul(tab[kJumpLo - 1], j, big);  // J^kJumpLo
    tab[kJumpLo] = tab[0];
    for (int a = 1; a < kJumpHi; ++a) gf2_mul(tab[kJumpLo + a - 1], big, tab[kJumpLo + a]);
    uint64_t *d = nullptr;
    const size_t bytes = tab.size() * sizeof(Gf2);
    if (cudaMalloc(&d, bytes) != cudaSuccess) return nullptr;
    if (cudaMemcpy(d, tab.data(), bytes, cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaFree(d);
        return nullptr;
    }
    g_jump[dev] = d;
    return d;
}

// Init blocks: kInitDraws draws (kInitDraws / 2 Box-Muller gaussians) per
// lane.  Table [2][256][4]: J = T^kInitDraws and J^32 (a warp's 32 blocks).
constexpr int kInitDraws = 32;
namespace {
std::mutex g_init_mu;
const uint64_t *g_init_jump[64] = {};
}  // namespace
const uint64_t *init_jump_table() {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_init_mu);
    if (dev < 0 || dev >= 64) return nullptr;
    if (g_init_jump[dev]) return g_init_jump[dev];
    std::vector<Gf2> tab(2);
    Gf2 t, tmp;
    gf2_step_matrix(t);
    tab[0] = t;  // T^32 by squaring (32 = 2^5)
    for (int k = 0; k < 5; ++k) {
        gf2_mul(tab[0], tab[0], tmp);
        tab[0] = tmp;
    }
    tab[1] = tab[0];  // (T^32)^32
    for (int k = 0; k < 5; ++k) {
        gf2_mul(tab[1], tab[1], tmp);
        tab[1] = tmp;
    }
    uint64_t *d = nullptr;
    const size_t bytes = tab.size() * sizeof(Gf2);
    if (cudaMalloc(&d, bytes) != cudaSuccess) return nullptr;
    if (cudaMemcpy(d, tab.data(), bytes, cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaFree(d);
        return nullptr;
    }
    g_init_jump[dev] = d;
    return d;
}

// s <- M s over GF(2) (M in row form, 256 x 4 u64)
__device__ __forceinline__ void gf2_apply(const uint64_t *__restrict__ m, Xoshiro &x) {
    uint64_t o[4] = {0, 0, 0, 0};
#pragma unroll 4
    for (int i = 0; i < 256; ++i) {
        const uint64_t *row = m + 4 * i;
        const uint64_t v = (__ldg(row) & x.s0) ^ (__ldg(row + 1) & x.s1) ^ (__ldg(row + 2) & x.s2) ^
                           (__ldg(row + 3) & x.s3);
        o[i >> 6] |= (uint64_t)(__popcll(v) & 1) << (i & 63);
    }
    x.s0 = o[0];
    x.s1 = o[1];
    x.s2 = o[2];
    x.s3 = o[3];
}
// Warp-cooperative y = M x (all 32 lanes, uniform x; every lane gets y):
// lane l takes rows l + 32 q (coalesced: the warp reads 1 KB of contiguous
// rows per q), each row's parity is a ballot bit, and row 64 w + 32 h + l is
// bit 32 h + l of word w.  Stepping one state through J = T^kJumpDraws this
// way replaces per-lane table jumps, whose lanes each walked a different
// 8 KB matrix (32 cache lines per load instruction, latency-bound chains).
__device__ __forceinline__ Xoshiro gf2_warp_apply(const uint64_t *M, const Xoshiro &x, int lane) {
    uint32_t m[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const uint64_t *row = M + 4 * (lane + 32 * q);
        const uint64_t v = (__ldg(row) & x.s0) ^ (__ldg(row + 1) & x.s1) ^ (__ldg(row + 2) & x.s2) ^
                           (__ldg(row + 3) & x.s3);
        m[q] = __ballot_sync(0xffffffffu, __popcll(v) & 1);
    }
    return Xoshiro(m[0] | ((uint64_t)m[1] << 32), m[2] | ((uint64_t)m[3] << 32), m[4] | ((uint64_t)m[5] << 32),
                   m[6] | ((uint64_t)m[7] << 32));
}
// advance x by `block` blocks of kJumpDraws draws
__device__ __forceinline__ void jump_blocks(const uint64_t *tab, int block, Xoshiro &x) {
    const int lo = block % kJumpLo, hi = block / kJumpLo;
    if (lo) gf2_apply(tab + (size_t)lo * 1024, x);
    if (hi) gf2_apply(tab + (size_t)(kJumpLo + hi) * 1024, x);
}

// ---------------------------------------------------------------- shuffle
// perm[net][epoch][n] (u16), Fisher-Yates of hybrid_nn.cpp:148-154 with
// Rng(substream_seed(shuffle_seed, epoch)) (:176).  One warp per (net,
// epoch): the n-1 draws below(i+1), i = n-1..1, are generated in blocks of
// kJumpDraws by the lanes in parallel (jump-ahead, bit-identical stream) into
// shared memory; lane 0 then applies the swap chain, which is inherently
// sequential, and the warp writes the permutation out.
constexpr int kPermWarps = 4;

__global__ void __launch_bounds__(32 * kPermWarps) perm_kernel(int n_nets, int epochs, int n,
                                                               const uint64_t *shuffle_seeds,
                                                               uint16_t *perm, const uint64_t *jtab) {
    extern __shared__ __align__(16) uint16_t sbuf[];  // per warp: idx[n8], draws[n8]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int job = blockIdx.x * kPermWarps + warp;
    if (job >= n_nets * epochs) return;  // warp-uniform
    const int net = job / epochs, epoch = job % epochs;
    const int n8 = (n + 7) & ~7;  // 16-byte aligned arrays
    uint16_t *idx = sbuf + (size_t)warp * 2 * n8, *jd = idx + n8;
    const Xoshiro r0(substream_seed(shuffle_seeds[net], (uint64_t)epoch));
    const int draws = n - 1, nblk = (draws + kJumpDraws - 1) / kJumpDraws;
    // block bk's state is J^bk r0 (J = lo[1] of the jump table): the warp steps
    // one state through J and lane t keeps the t-th of each 32
    Xoshiro x = r0;
    for (int base = 0; base < nblk; base += 32) {
        Xoshiro r = x;
        for (int t = 0; t < 32 && base + t < nblk; ++t) {
            if (lane == t) r = x;
            x = gf2_warp_apply(jtab + 1024, x, lane);
        }
        const int bk = base + lane;
        if (bk >= nblk) continue;
        const int k_end = min(draws, (bk + 1) * kJumpDraws);
        for (int k = bk * kJumpDraws; k < k_end; ++k) {  // draw k is for i = n-1-k
            const int i = n - 1 - k;
            jd[k] = (uint16_t)r.below((uint64_t)i + 1);
        }
    }
    for (int i = lane; i < n; i += 32) idx[i] = (uint16_t)i;
    __syncwarp();
    if (lane == 0) {
        // the draws are read eight at a time, one group ahead: loaded inside
        // the chain they would wait behind the previous swap's stores (same
        // shared array), doubling the per-step latency
        auto swap = [&](int k, uint32_t j) {
            const int i = n - 1 - k;
            const uint16_t t = idx[i];
            idx[i] = idx[j];
            idx[j] = t;
        };
        const uint4 *jd4 = reinterpret_cast<const uint4 *>(jd);
        const int full = draws >> 3;
        uint4 q = full > 0 ? jd4[0] : make_uint4(0, 0, 0, 0);
        for (int g = 0; g < full; ++g) {
            const uint4 cur = q;
            if (g + 1 < full) q = jd4[g + 1];
            const uint32_t w[4] = {cur.x, cur.y, cur.z, cur.w};
#pragma unroll
            for (int e = 0; e < 8; ++e) swap(8 * g + e, (w[e >> 1] >> (16 * (e & 1))) & 0xFFFFu);
        }
        for (int k = 8 * full; k < draws; ++k) swap(k, jd[k]);
    }
    __syncwarp();
    uint16_t *out = perm + (size_t)job * n;
    for (int i = lane; i < n; i += 32) out[i] = idx[i];
}

// Throughput form: one thread per (net, epoch) with its own sequential
// stream and index array -- the right shape when there are many more
// shuffles than SMs x warps (the swap chains then fill the machine).  The
// finished arrays leave through the warp: for each of its 32 jobs the lanes
// store consecutive 32-bit words, so every store instruction is one coalesced
// line instead of 32 scattered 2-byte writes (the scattered form was L2
// transaction bound: ~70 ms per C5 chunk).
__global__ void perm_thread_kernel(int n_nets, int epochs, int n, const uint64_t *shuffle_seeds,
                                   uint16_t *perm) {
    extern __shared__ __align__(16) uint16_t sidx[];
    const int lane = threadIdx.x & 31;
    const int np = (n + 1) & ~1;  // per-thread array stride: whole 32-bit words
    uint16_t *idx = sidx + (size_t)threadIdx.x * np;
    const int jobs = n_nets * epochs;
    const int warps_total = gridDim.x * (blockDim.x >> 5);
    for (int base = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; base < jobs;
         base += warps_total * 32) {
        const int job = base + lane;
        if (job < jobs) {
            const int net = job / epochs, epoch = job % epochs;
            for (int i = 0; i < n; ++i) idx[i] = (uint16_t)i;
            Xoshiro r(substream_seed(shuffle_seeds[net], (uint64_t)epoch));
            for (int i = n - 1; i > 0; --i) {
                const int j = (int)r.below((uint64_t)i + 1);
                const uint16_t t = idx[i];
                idx[i] = idx[j];
                idx[j] = t;
            }
        }
        __syncwarp();
        const int nj = min(32, jobs - base);
        const uint16_t *wbase = sidx + (size_t)(threadIdx.x & ~31) * np;
        for (int t = 0; t < nj; ++t) {
            const uint16_t *src = wbase + (size_t)t * np;
            uint16_t *dst = perm + (size_t)(base + t) * n;
            // dst is 4-byte aligned when (base + t) * n is even
            if ((((size_t)(base + t) * n) & 1) == 0) {
                const uint32_t *s32 = reinterpret_cast<const uint32_t *>(src);
                uint32_t *d32 = reinterpret_cast<uint32_t *>(dst);
                for (int w = lane; w < n / 2; w += 32) d32[w] = s32[w];
                if ((n & 1) && lane == 0) dst[n - 1] = src[n - 1];
            } else {
                for (int i = lane; i < n; i += 32) dst[i] = src[i];
            }
        }
        __syncwarp();
    }
}

int perm_launch(int n_nets, int epochs, int n, const uint64_t *seeds, uint16_t *perm,
                cudaStream_t st, int max_tpb) {
    if (n > 65535) return NOMA_ERR_UNSUPPORTED;
    const int jobs = n_nets * epochs;
    if (jobs == 0 || n < 1) return NOMA_OK;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // many shuffles: thread per job, whole warps of index arrays in shared
    // memory (max_tpb 32: one warp, 88 KB at n = 1370, one CTA per SM -- the
    // form that can sit beside two training CTAs in the overlapped pipeline)
    const int np = (n + 1) & ~1;
    int tpb = (int)((200 * 1024) / (2 * (size_t)np));
    tpb = (tpb > max_tpb ? max_tpb : tpb) & ~31;
    if (jobs > 16 * sms && tpb >= 32) {
        const size_t smem = (size_t)tpb * np * sizeof(uint16_t);
        cudaFuncSetAttribute(perm_thread_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int grid = max_tpb < 64 ? sms : (jobs + tpb - 1) / tpb;
        perm_thread_kernel<<<grid, tpb, smem, st>>>(n_nets, epochs, n, seeds, perm);
        return cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;
    }
    if ((n - 1 + kJumpDraws - 1) / kJumpDraws > kJumpLo * kJumpHi) return NOMA_ERR_UNSUPPORTED;
    const uint64_t *jt = jump_table();
    if (!jt) return NOMA_ERR_CUDA;
    const size_t smem = (size_t)kPermWarps * 2 * ((n + 7) & ~7) * sizeof(uint16_t);
    if (smem > 227 * 1024) return NOMA_ERR_UNSUPPORTED;
    cudaFuncSetAttribute(perm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    perm_kernel<<<(jobs + kPermWarps - 1) / kPermWarps, 32 * kPermWarps, smem, st>>>(n_nets, epochs, n,
                                                                                    seeds, perm, jt);
    return cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;
}

// ------------------------------------------------------------------- init
// He-normal initialisation (hybrid_nn.cpp:43-52), one CTA per net.  The
// reference stream (2 u64 per gaussian, row-major per layer) is cut into
// blocks of kJumpDraws draws; thread b jumps its own xoshiro copy to block b
// (jump_blocks) and turns the block's 64 pairs into Box-Muller draws (the FP64
// log/sqrt/cos dominate), scattered into the plan (FP32, FusedPlan layout)
// and/or the flat FP64 parameter vector.  Seeds come from `seeds`
// (Rng(seed)) or, when `states` is non-null, from caller xoshiro states that
// are advanced in place past all draws (init_params(..., Rng&)).
constexpr int kInitThreads = 512;  // 16 warps: a [32, 64, 64] net's 12 chunks of 32 blocks run at once

__global__ void __launch_bounds__(kInitThreads) init_block_kernel(
    NetGeom g, const uint64_t *seeds, uint64_t *states, const double *w0, bool keep_w0, float *plans,
    double *theta, int ptrain, const uint64_t *jtab) {
    const int net = blockIdx.x, tid = threadIdx.x;
    float *pl = plans ? plans + (size_t)net * g.plan_total : nullptr;
    double *th = theta ? theta + (size_t)net * ptrain : nullptr;
    // zero outputs, w0 slot (unless a concurrent LLS writes it: keep_w0),
    // biases / final (theta)
    if (pl) {
        for (int i = tid + (keep_w0 ? g.dims[0] : 0); i < g.plan_total; i += kInitThreads) pl[i] = 0.0f;
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
    const Xoshiro r0 = states ? Xoshiro(states[net * 4], states[net * 4 + 1], states[net * 4 + 2], states[net * 4 + 3])
                              : Xoshiro(seeds[net]);
    // every thread holds the caller's state before the last block's lane
    // writes the advanced state back over it
    __syncthreads();
    constexpr int G = kInitDraws / 2;  // gaussians per block (lane)
    const int blocks = (total + G - 1) / G;
    // chunks of 32 blocks per warp: the chunk's first state by c steps of
    // J^32 (jtab[1]), then the warp steps through J (jtab[0]) and lane t keeps
    // block 32 c + t (gf2_warp_apply).  16 gaussians per lane: a C1 net's
    // 2048 draws take four warps instead of one (Box-Muller is the long part)
    const int warp = tid >> 5, lane = tid & 31;
    for (int c = warp; 32 * c < blocks; c += kInitThreads / 32) {
        Xoshiro x = r0;
        for (int i = 0; i < c; ++i) x = gf2_warp_apply(jtab + 1024, x, lane);
        Xoshiro r = x;
        for (int t = 0; t < 32 && 32 * c + t < blocks; ++t) {
            if (lane == t) r = x;
            x = gf2_warp_apply(jtab, x, lane);
        }
        const int b = 32 * c + lane;
        if (b >= blocks) continue;
        const int w_end = min(total, (b + 1) * G);
        int l = 1;
        for (int w = b * G; w < w_end; ++w) {
            const uint64_t a1 = r.next(), a2 = r.next();
            while (w >= start[l + 1]) ++l;
            const int fan_in = g.dims[l - 1];
            const int off = w - start[l], row = off / fan_in, col = off % fan_in;
            // Box-Muller cosine half (rng.hpp:58-62)
            const double u1 = 1.0 - static_cast<double>(a1 >> 11) * 0x1.0p-53;
            const double u2 = static_cast<double>(a2 >> 11) * 0x1.0p-53;
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
        if (states && w_end == total) {  // the last block leaves the stream past every draw
            states[net * 4] = r.s0;
            states[net * 4 + 1] = r.s1;
            states[net * 4 + 2] = r.s2;
            states[net * 4 + 3] = r.s3;
        }
    }
}

int init_state_launch(const NetGeom &g, int n_nets, uint64_t *states, const double *w0,
                      float *plans, double *theta, int ptrain, cudaStream_t st) {
    if (n_nets == 0) return NOMA_OK;
    const uint64_t *jt = init_jump_table();
    if (!jt) return NOMA_ERR_CUDA;
    init_block_kernel<<<n_nets, kInitThreads, 0, st>>>(g, nullptr, states, w0, false, plans, theta, ptrain, jt);
    return cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;
}

int init_launch(const NetGeom &g, int n_nets, const uint64_t *seeds, const double *w0, bool keep_w0,
                float *plans, cudaStream_t st) {
    if (n_nets == 0) return NOMA_OK;
    const uint64_t *jt = init_jump_table();
    if (!jt) return NOMA_ERR_CUDA;
    init_block_kernel<<<n_nets, kInitThreads, 0, st>>>(g, seeds, nullptr, w0, keep_w0, plans, nullptr, 0, jt);
    return cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;
}

int init_theta_launch(const NetGeom &g, int n_nets, const uint64_t *seeds, double *theta, int ptrain,
                      cudaStream_t st) {
    if (n_nets == 0) return NOMA_OK;
    const uint64_t *jt = init_jump_table();
    if (!jt) return NOMA_ERR_CUDA;
    init_block_kernel<<<n_nets, kInitThreads, 0, st>>>(g, seeds, nullptr, nullptr, false, nullptr, theta, ptrain, jt);
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
        if (p.data_rx64) {
            double *o = p.data_rx64 + (((size_t)s * p.ND + td) * p.M + m) * 2;
            o[0] = re;
            o[1] = im;
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
