// Data-phase detection on the 5th-generation tensor cores (tcgen05, sm_100a):
// hybrid_nn::detect (hybrid_nn.cpp:197-199) / fused_forward_f32
// (fused_inference.cpp:222-231) with hard_decision_qpsk and bit_error_rate
// (eval.cpp:38-65) fused into the epilogue.
//
// Precision: every layer contraction is 3xTF32 -- x = x_hi + x_lo with x_hi
// the TF32 truncation of x and x_lo = x - x_hi (exact in FP32), and
// A B ~ A_hi B_hi + A_hi B_lo + A_lo B_hi accumulated in FP32 in TMEM.  The
// dropped A_lo B_lo term is ~2^-22 relative, so soft outputs stay at FP32
// level and the hard decisions match the FFMA path (the north star's gate
// for using tensor cores on the data phase).
//
// Per CTA: one user network, one CTA per SM, a persistent warp-specialised
// pipeline over 128-row tiles (64 QPSK symbols); see detect_ws_kernel below.
// Each tile's widened rows (row 2s = [Re x_s; Im x_s], 2s+1 = [Im x_s;
// -Re x_s], iq_transform.cpp:17-20) are formed straight from the complex
// samples and stored hi/lo in the no-swizzle K-major core-matrix layout
// (8 rows x 16 B per core matrix); tcgen05.mma kind::tf32 (M=128) runs the
// hidden layers with FP32 accumulators in TMEM; the epilogues add the bias,
// apply ReLU, stage the next layer's A operand in TMEM (tcgen05.st) or form
// yhat = x.w0 + a_N . w_final; lane pairs (2s, 2s+1) give Re/Im of symbol s,
// whose sign bits are the QPSK decision (ties -> 0); errors against the truth
// codes are warp-reduced into one atomic per warp.
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"

namespace noma_dev {

namespace {

constexpr int kTcRows = 128;  // rows per tile = TMEM lanes = M of every MMA

__device__ __forceinline__ uint32_t tc_s2u(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// shared-memory matrix descriptor, no swizzle, K-major core matrices:
// lbo = byte stride between core matrices along K, sbo = along M/N
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm100)
    return d;
}
// instruction descriptor: D f32, A/B tf32, both K-major, M = 128
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(ad), "l"(bd), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint32_t mbar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar)
                 : "memory");
}
// the suspend-time hint lets a waiting warp sleep until the phase completes
// instead of re-polling (the pipeline roles spend much of their time here)
__device__ __forceinline__ void tc_mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\nTCW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n\t@!p bra TCW_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// tcgen05.ld without the wait: several loads in flight, one tmem_wait_ld()
__device__ __forceinline__ void tmem_ld16_nw(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// 16 columns of this thread's TMEM lane (the layer-2 A operand row)
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
        "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
        "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
        "r"(__float_as_uint(v[15])));
}
// A operand from TMEM (a_tmem: column address of the K-step), B from smem
__device__ __forceinline__ void umma_tf32_ta(uint32_t tmem_d, uint32_t a_tmem, uint64_t bd, uint32_t idesc,
                                             uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(a_tmem), "l"(bd), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }
// packed FP32x2 arithmetic (sm_100a FADD2 / FFMA2): per lane identical to the
// scalar operation, half the instructions
typedef unsigned long long p2_t;
__device__ __forceinline__ p2_t pk2(float a, float b) {
    p2_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float2 up2(p2_t v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
__device__ __forceinline__ p2_t add2(p2_t a, p2_t b) {
    p2_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ p2_t sub2(p2_t a, p2_t b) {
    p2_t d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ p2_t fma2(p2_t a, p2_t b, p2_t c) {
    p2_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ p2_t relu2(p2_t v) {
    const float2 f = up2(v);
    return pk2(fmaxf(f.x, 0.f), fmaxf(f.y, 0.f));
}

// byte offset of element (row r, k) in a K-major no-swizzle operand with
// `kb` 4-element k-blocks per row group: core (r/8, k/4) at
// ((r/8) * kb + k/4) * 128 B, (r%8) * 16 B + (k%4) * 4 B inside it
__device__ __forceinline__ int core_off(int r, int k, int kb) {
    return (((r >> 3) * kb + (k >> 2)) << 7) + ((r & 7) << 4) + ((k & 3) << 2);
}
// store a 4-float k-block of row r (hi and lo planes)
__device__ __forceinline__ void put4(char *hi, char *lo, int r, int k, int kb, float4 v) {
    const float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
    const int o = core_off(r, k, kb);
    *reinterpret_cast<float4 *>(hi + o) = h;
    const float2 l01 = up2(sub2(pk2(v.x, v.y), pk2(h.x, h.y))), l23 = up2(sub2(pk2(v.z, v.w), pk2(h.z, h.w)));
    *reinterpret_cast<float4 *>(lo + o) = make_float4(l01.x, l01.y, l23.x, l23.y);
}

}  // namespace

struct DetectTcParams {
    NetGeom g;
    int n_nets, K, rows, tiles;  // rows = data symbols per slot; tiles of 64 symbols
    int stride;                  // row stride of data / truth / soft / codes
    const float *data;           // [S][rows][M] complex f32
    const float *plans;
    const uint8_t *truth;        // [S][rows][K] codes, nullable
    float *soft;                 // [net][rows] complex, nullable
    uint8_t *codes;              // [net][rows], nullable
    uint32_t *errors;            // [net], nullable
    uint32_t *sym_errors;        // [net], nullable
    const int *status;
    long long *clocks;           // NOMA_DETECT_CLK: per-role cycles of CTA (0, 0), nullable
};

// W0 = input width 2M, H = hidden width, NL = hidden layers (1 or 2).
// ---------------------------------------------------------------------------
// Warp-specialised pipeline (one CTA per SM, persistent over the net's tiles):
//   warps 0-3    loaders: thread r forms widened row r of a tile from global
//                samples, computes the linear branch lin = x . w0 in FP32, and
//                stages the row hi/lo as the layer-1 A operand of slot
//                (tile parity): in TMEM with tcgen05.st for a 32-wide input,
//                in smem (K-major core layout) for a 64-wide one; lin goes to
//                an 8-slot smem ring;
//   warps 4-7    epilogue 1: D[slot] -> a1 = relu(D + b1), split hi/lo into
//                TMEM A2[slot] (the layer-2 A operand); with one hidden layer
//                the output directly;
//   warps 8-11   epilogue 2 (two layers): D[slot] -> yhat = lin + a2 . w ->
//                QPSK decision and bit errors;
//   next 2 warps issue the layer-1 tcgen05.mma chains of even / odd tiles;
//   last 2 warps issue the layer-2 chains of even / odd tiles.
// Every hand-off is an mbarrier with one arrival per producing warp; MMA
// completion by tcgen05.commit.  TMEM (512 columns): D[2] at 0 / 64 -- the
// layer-2 accumulator reuses its slot's layer-1 columns, which epilogue 1 has
// drained before it releases A2, and the next layer-1 MMA into the slot waits
// for the final epilogue; A2[2] (hi, lo) at 128 / 256; A1[2] (hi, lo) at
// 384 / 448 for a 32-wide input.
// Why (tools/microbench/umma_rate.cu, tmem_bw.cu, NOMA_DETECT_CLK): an M=128,
// N=64 tf32 MMA reaches the 32-cycle pipe floor only with A in TMEM and two
// concurrent issuers (one issuer: ~47 cycles; A in smem: ~48 cycles, bound by
// the smem operand read); TMEM loads/stores are cheap (~300-800 B/cycle), and
// shared memory is the contended resource -- while the tensor core streams
// operands from it, epilogue LDS / mbarrier latency grows ~10x.
template <int W0, int NL>
struct WsRoles {
    static constexpr bool kA1Tmem = W0 <= 32;            // layer-1 A operand in TMEM
    static constexpr int kMma1Warp = NL > 1 ? 12 : 8;    // layer-1 issuers: kMma1Warp, +1
    static constexpr int kMma2Warp = kMma1Warp + 2;      // layer-2 issuers (two layers): +0, +1
    static constexpr int kWarps = NL > 1 ? 16 : 10;
    static constexpr int kThreads = 32 * kWarps;
};
// lin = x . w0 travels from the loaders to the last stage through a ring of
// kLinSlots slots: with only two, the loaders would be held to within two
// tiles of the final epilogue and starve the whole pipeline
constexpr int kLinSlots = 8;
// A2Full is per (slot, column half): layer 2's first four k-steps read only
// columns 0-31 of A2, so they start while epilogue 1 still works on 32-63
enum WsBar { kA1Full = 0, kM1Done = 2, kDEmpty = 4, kA2Full = 6, kM2Done = 10, kLinFull = 12,
             kLinEmpty = 12 + kLinSlots, kWsBars = 12 + 2 * kLinSlots };

// one arrival per warp (barrier count = 4 warps per role): 128 per-thread
// arrivals on one mbarrier serialise.  __syncwarp orders the lanes' prior
// shared-memory / tcgen05 writes (each lane has fenced them) before lane 0's
// release-arrive.
__device__ __forceinline__ void ws_arrive(uint32_t bar) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// per-thread arrival (barrier count 128) for the x . w0 ring, whose payload is
// ordinary shared memory: compute-sanitizer racecheck does not credit
// __syncwarp's memory ordering to a lane-0 arrival
// (tools/microbench/warp_arrive_repro.cu), so this hand-off stays per lane
__device__ __forceinline__ void ws_arrive_lane(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

template <int W0, int H, int NL>
constexpr size_t detect_ws_smem() {
    return 2 * (size_t)H * W0 * 4 + (NL > 1 ? 2 * (size_t)H * H * 4 : 0) +
           (WsRoles<W0, NL>::kA1Tmem ? 0 : 4 * (size_t)kTcRows * W0 * 4) + (size_t)(NL + 1) * H * 4 +
           (size_t)W0 * 4 + kLinSlots * kTcRows * 4 + 8 * kWsBars + 16;
}

template <int W0, int H, int NL>
__global__ void __launch_bounds__(WsRoles<W0, NL>::kThreads, 1) detect_ws_kernel(DetectTcParams p) {
    using R = WsRoles<W0, NL>;
    constexpr bool kA1T = R::kA1Tmem;
    constexpr int M = W0 / 2;
    constexpr int KB0 = W0 / 4, KBH = H / 4;  // k-blocks per row group
    constexpr uint32_t A1B = kTcRows * W0 * 4, B1B = H * W0 * 4, B2B = H * H * 4;
    constexpr uint32_t kD = 0, kA2 = 128, kA2S = 128, kA1 = 384, kA1S = 64;  // TMEM columns
    static_assert(H == 64, "TMEM column plan assumes 64-wide hidden layers");
    extern __shared__ __align__(1024) char smem[];
    char *b1h = smem, *b1l = b1h + B1B;
    char *b2h = b1l + B1B, *b2l = b2h + (NL > 1 ? B2B : 0);
    char *a1 = b2l + (NL > 1 ? B2B : 0);                                 // smem A1 [slot][hi | lo] (W0 = 64)
    float *bias = reinterpret_cast<float *>(a1 + (kA1T ? 0 : 4 * A1B));  // [NL][H]
    float *wf = bias + NL * H;                                           // [H]
    float *w0s = wf + H;                                                 // [W0]
    float *lin_s = w0s + W0;                                             // [kLinSlots][128]
    uint64_t *bars = reinterpret_cast<uint64_t *>(lin_s + kLinSlots * kTcRows);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + kWsBars);
    auto bar = [&](int i) { return tc_s2u(bars + i); };
    // NOMA_DETECT_CLK: lane 0 of each role's first warp in CTA (0, 0) records
    // [total loop cycles, cycles waiting at site 0, at site 1, TMEM loads, dot,
    // emit] per role (roles: loaders, epilogue 1, epilogue 2, then one per
    // issuing warp)
    const int role = (threadIdx.x >> 7) < 3 ? (int)(threadIdx.x >> 7) : 3 + (int)(threadIdx.x >> 5) - 12;
    long long *ck = NOMA_PROBE_ON(p.clocks && blockIdx.x == 0 && (threadIdx.x & (threadIdx.x < 384 ? 127 : 31)) == 0)
                        ? p.clocks + 6 * role
                        : nullptr;
    // accumulated in shared memory: a global += per tile would distort the stage
    __shared__ long long ck_s[8 * 6];
    long long *cv = ck ? ck_s + 6 * role : nullptr;
    if (cv)
        for (int c = 0; c < 6; ++c) cv[c] = 0;
    auto wait = [&](int site, uint32_t b, uint32_t ph) {
        if (ck) {
            const long long t0 = clock64();
            tc_mbar_wait(b, ph);
            cv[1 + site] += clock64() - t0;
        } else {
            tc_mbar_wait(b, ph);
        }
    };
    const long long tstart = ck ? clock64() : 0;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const NetGeom &g = p.g;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(tc_s2u(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 32) {
        for (int i = 0; i < kWsBars; ++i) {
            const bool commit = (i >= kM1Done && i < kM1Done + 2) || (i >= kM2Done && i < kM2Done + 2);
            const bool lin = i >= kLinFull;  // x . w0 ring: per-thread arrivals
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar(i)),
                         "r"(commit ? 1 : lin ? kTcRows : kTcRows / 32));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;
    // launched as a programmatic dependent of the training kernel: the plans
    // it writes are read below (a no-op for an ordinary launch)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // this CTA's share of the global (net, tile) range; one pipeline segment
    // per net it touches, the mbarrier phases running on across segments (ib)
    const long long T = (long long)p.n_nets * p.tiles;
    const long long t_lo = T * blockIdx.x / gridDim.x, t_hi = T * (blockIdx.x + 1) / gridDim.x;
    int net = 0, d = 0, k = 0, first = 0, ntile = 0, ib = 0;
    // decision + bit errors of widened row r (lane pairs = Re/Im of a symbol)
    uint32_t my_err = 0, my_ser = 0;
    auto emit = [&](int tile, int r, float y, uint8_t truth) {
        const float yo = __shfl_xor_sync(0xffffffffu, y, 1);
        const int s = tile * 64 + (r >> 1);
        if (!(r & 1) && s < p.rows) {
            const uint8_t code = (uint8_t)((y < 0.f ? 1 : 0) | (yo < 0.f ? 2 : 0));  // eval.cpp:41-42
            if (p.codes) p.codes[(size_t)net * p.stride + s] = code;
            if (p.soft) *reinterpret_cast<float2 *>(p.soft + ((size_t)net * p.stride + s) * 2) = make_float2(y, yo);
            if (p.truth) {
                const uint32_t e = __popc((unsigned)(truth ^ code) & 3u);
                my_err += e;
                my_ser += e ? 1u : 0u;
            }
        }
    };
    auto truth_of = [&](int tile, int r) -> uint8_t {
        const int s = tile * 64 + (r >> 1);
        return p.truth && !(r & 1) && s < p.rows ? p.truth[((size_t)d * p.stride + s) * p.K + k] : (uint8_t)0;
    };
    // sum_c relu(v_c + b_c) w_c over 16 columns
    // (partials: acc2[0] = columns 4j, 4j+1; acc2[1] = 4j+2, 4j+3)
    auto dot16 = [&](const uint32_t (&v)[16], const float *b, const float *w, p2_t (&acc2)[2]) {
#pragma unroll
        for (int q = 0; q < 16; q += 4) {
            const float4 b4 = *reinterpret_cast<const float4 *>(b + q);
            const float4 w4 = *reinterpret_cast<const float4 *>(w + q);
            const p2_t a01 = relu2(add2(pk2(__uint_as_float(v[q]), __uint_as_float(v[q + 1])), pk2(b4.x, b4.y)));
            const p2_t a23 = relu2(add2(pk2(__uint_as_float(v[q + 2]), __uint_as_float(v[q + 3])), pk2(b4.z, b4.w)));
            acc2[0] = fma2(a01, pk2(w4.x, w4.y), acc2[0]);
            acc2[1] = fma2(a23, pk2(w4.z, w4.w), acc2[1]);
        }
    };
    // the final stage: D[slot] (drained) + lin -> decision (epilogue 1 or 2)
    auto finish = [&](int i, int tile, int r, const uint32_t (&v)[H / 16][16], const float *bN, uint8_t truth) {
        const int ls = i % kLinSlots;
        wait(1, bar(kLinFull + ls), (i / kLinSlots) & 1);
        const float lin = lin_s[ls * kTcRows + r];
        ws_arrive_lane(bar(kLinEmpty + ls));
        const long long td0 = ck ? clock64() : 0;
        p2_t acc2[2] = {0ull, 0ull};
#pragma unroll
        for (int c = 0; c < H / 16; ++c) dot16(v[c], bN + 16 * c, wf + 16 * c, acc2);
        const float2 s01 = up2(acc2[0]), s23 = up2(acc2[1]);
        const float y = lin + ((s01.x + s01.y) + (s23.x + s23.y));  // hybrid_nn.cpp:81
        const long long td1 = ck ? clock64() : 0;
        emit(tile, r, y, truth);
        if (ck) {
            cv[4] += td1 - td0;
            cv[5] += clock64() - td1;
        }
    };
    // drain D[slot] of tile i into registers and release the slot / columns
    auto drain = [&](uint32_t col, uint32_t trow, uint32_t (&v)[H / 16][16]) {
        const long long tl0 = ck ? clock64() : 0;
#pragma unroll
        for (int c = 0; c < H / 16; ++c) tmem_ld16_nw(trow + col + 16 * c, v[c]);
        tmem_wait_ld();
        if (ck) cv[3] += clock64() - tl0;
        asm volatile("tcgen05.fence::before_thread_sync;");
    };

    for (long long t0 = t_lo; t0 < t_hi; t0 += ntile) {
    net = (int)(t0 / p.tiles);
    first = (int)(t0 - (long long)net * p.tiles);
    ntile = (int)((t_hi < (long long)(net + 1) * p.tiles ? t_hi : (long long)(net + 1) * p.tiles) - t0);
    d = net / p.K;
    k = net % p.K;
    if (p.status && p.status[net] != NOMA_OK) {
        if (first == 0 && threadIdx.x == 0 && p.errors) p.errors[net] = 0xFFFFFFFFu;
        if (first == 0 && threadIdx.x == 0 && p.sym_errors) p.sym_errors[net] = 0xFFFFFFFFu;
        continue;
    }
    // ---- the net's weights: hi/lo planes in the K-major core layout (FusedPlan
    // order); the previous segment's MMAs have all completed (every one was
    // waited on by an epilogue before the closing barrier)
    const float *pl = p.plans + (size_t)net * g.plan_total;
    for (int i = threadIdx.x; i < H * KB0; i += R::kThreads) {
        const int j = i / KB0, kq = (i - j * KB0) * 4;
        put4(b1h, b1l, j, kq, KB0, *reinterpret_cast<const float4 *>(pl + g.plan_w[1] + j * g.plan_pad[0] + kq));
    }
    if constexpr (NL > 1) {
        for (int i = threadIdx.x; i < H * KBH; i += R::kThreads) {
            const int j = i / KBH, kq = (i - j * KBH) * 4;
            put4(b2h, b2l, j, kq, KBH, *reinterpret_cast<const float4 *>(pl + g.plan_w[2] + j * g.plan_pad[1] + kq));
        }
    }
    for (int i = threadIdx.x; i < NL * H; i += R::kThreads) bias[i] = pl[g.plan_b[1 + i / H] + i % H];
    for (int i = threadIdx.x; i < H; i += R::kThreads) wf[i] = pl[g.plan_f + i];
    for (int i = threadIdx.x; i < W0; i += R::kThreads) w0s[i] = pl[g.plan_w0 + i];
    // the weight planes are read by the tensor core (async proxy)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (warp < 4) {
        // ---------------- loaders: widened rows -> A1[slot] (hi/lo), lin ---------
        const int r = threadIdx.x, sym = r >> 1;
        const bool odd = r & 1;
        const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
        const float2 *src = reinterpret_cast<const float2 *>(p.data) + (size_t)d * p.stride * M;
        float2 xs[M];
        auto load = [&](int tile) {
            const int s = tile * 64 + sym;
            const bool ok = s < p.rows;
#pragma unroll
            for (int m = 0; m < M; m += 2) {
                const float4 v = ok ? *reinterpret_cast<const float4 *>(src + (size_t)s * M + m)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
                xs[m] = make_float2(v.x, v.y);
                xs[m + 1] = make_float2(v.z, v.w);
            }
        };
        load(first);
        for (int j = 0; j < ntile; ++j) {
            const int i = ib + j;
            const int sl = i & 1;
            const uint32_t ph = (i >> 1) & 1;
            p2_t l2[2] = {0ull, 0ull};  // x . w0 (hybrid_nn.cpp:81, linear branch), 4 partials
            wait(0, bar(kM1Done + sl), ph ^ 1);  // A1[sl] read by tile i-2's MMAs
            asm volatile("tcgen05.fence::after_thread_sync;");
            float rh[kA1T ? W0 : 1], rl[kA1T ? W0 : 1];  // the row, hi / lo (TMEM staging)
            (void)rh;
            (void)rl;
#pragma unroll
            for (int m = 0; m < M; m += 4) {
                const float4 re = make_float4(xs[m].x, xs[m + 1].x, xs[m + 2].x, xs[m + 3].x);
                const float4 im = make_float4(xs[m].y, xs[m + 1].y, xs[m + 2].y, xs[m + 3].y);
                // widened row (iq_transform.cpp:17-20): [Re; Im] or [Im; -Re]
                const float4 lo4 = odd ? im : re;
                const float4 hi4 = odd ? make_float4(-re.x, -re.y, -re.z, -re.w) : im;
                if constexpr (kA1T) {
                    const float v8[8] = {lo4.x, lo4.y, lo4.z, lo4.w, hi4.x, hi4.y, hi4.z, hi4.w};
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const int kk = e < 4 ? m + e : M + m + e - 4;
                        rh[kk] = tf32_hi(v8[e]);
                        rl[kk] = v8[e] - rh[kk];
                    }
                } else {
                    char *ah = a1 + sl * 2 * A1B, *al = ah + A1B;
                    put4(ah, al, r, m, KB0, lo4);
                    put4(ah, al, r, M + m, KB0, hi4);
                }
                const float4 wa = *reinterpret_cast<const float4 *>(w0s + m);
                const float4 wb = *reinterpret_cast<const float4 *>(w0s + M + m);
                l2[0] = fma2(pk2(lo4.x, lo4.y), pk2(wa.x, wa.y), l2[0]);
                l2[1] = fma2(pk2(lo4.z, lo4.w), pk2(wa.z, wa.w), l2[1]);
                l2[0] = fma2(pk2(hi4.x, hi4.y), pk2(wb.x, wb.y), l2[0]);
                l2[1] = fma2(pk2(hi4.z, hi4.w), pk2(wb.z, wb.w), l2[1]);
            }
            if constexpr (kA1T) {
#pragma unroll
                for (int c = 0; c < W0 / 16; ++c) {
                    float h16[16], l16[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        h16[e] = rh[16 * c + e];
                        l16[e] = rl[16 * c + e];
                    }
                    tmem_st16(trow + kA1 + sl * kA1S + 16 * c, h16);
                    tmem_st16(trow + kA1 + sl * kA1S + W0 + 16 * c, l16);
                }
            }
            if (j + 1 < ntile) load(first + j + 1);  // in flight until the next stage
            if constexpr (kA1T) {
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;");
            } else {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            }
            ws_arrive(bar(kA1Full + sl));
            const int ls = i % kLinSlots;
            wait(1, bar(kLinEmpty + ls), ((i / kLinSlots) & 1) ^ 1);
            const float2 q01 = up2(l2[0]), q23 = up2(l2[1]);
            lin_s[ls * kTcRows + r] = (q01.x + q01.y) + (q23.x + q23.y);
            ws_arrive_lane(bar(kLinFull + ls));
        }
    } else if (warp < 8) {
        // ---------------- epilogue 1 --------------------------------------------
        const int q = warp - 4, r = q * 32 + lane;
        const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
        // truth codes two tiles ahead (a global load per tile would otherwise
        // sit exposed on this stage's critical path)
        uint8_t tq0 = NL == 1 ? truth_of(first, r) : 0, tq1 = NL == 1 ? truth_of(first + 1, r) : 0;
        for (int j = 0; j < ntile; ++j) {
            const int i = ib + j;
            const int sl = i & 1;
            const uint32_t ph = (i >> 1) & 1;
            uint8_t truth = 0;
            if constexpr (NL == 1) {
                truth = tq0;
                tq0 = tq1;
                tq1 = truth_of(first + j + 2, r);
            }
            wait(0, bar(kM1Done + sl), ph);
            asm volatile("tcgen05.fence::after_thread_sync;");
            uint32_t v1[H / 16][16];
            // two layers: the layer-1 accumulator lives in A2[sl]'s hi half
            drain(NL > 1 ? kA2 + sl * kA2S : kD + sl * H, trow, v1);
            if constexpr (NL == 1) {
                ws_arrive(bar(kDEmpty + sl));
                finish(i, first + j, r, v1, bias, truth);
            } else {
                // A2[sl] is free once tile i-2's layer-2 MMAs are done
                wait(1, bar(kM2Done + sl), ph ^ 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t a2 = trow + kA2 + sl * kA2S;
                long long te0 = ck ? clock64() : 0;
#pragma unroll
                for (int c = 0; c < H / 16; ++c) {
                    if (ck && c == 2) te0 = clock64();
                    float hi[16], lo[16];
#pragma unroll
                    for (int e4 = 0; e4 < 16; e4 += 4) {
                        const float4 b4 = *reinterpret_cast<const float4 *>(bias + 16 * c + e4);
#pragma unroll
                        for (int e = 0; e < 4; e += 2) {
                            const p2_t a = relu2(add2(pk2(__uint_as_float(v1[c][e4 + e]), __uint_as_float(v1[c][e4 + e + 1])),
                                                      e ? pk2(b4.z, b4.w) : pk2(b4.x, b4.y)));
                            const float2 af = up2(a);
                            hi[e4 + e] = tf32_hi(af.x);
                            hi[e4 + e + 1] = tf32_hi(af.y);
                            const float2 lf = up2(sub2(a, pk2(hi[e4 + e], hi[e4 + e + 1])));
                            lo[e4 + e] = lf.x;
                            lo[e4 + e + 1] = lf.y;
                        }
                    }
                    tmem_st16(a2 + 16 * c, hi);
                    tmem_st16(a2 + H + 16 * c, lo);
                    if (c % 2 == 1) {  // a column half of A2 (hi and lo) is in TMEM
                        const long long te1 = ck ? clock64() : 0;
                        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                        asm volatile("tcgen05.fence::before_thread_sync;");
                        if (ck) {  // epilogue 1: [4] compute + store issue, [5] store wait
                            cv[4] += te1 - te0;
                            cv[5] += clock64() - te1;
                        }
                        ws_arrive(bar(kA2Full + 2 * sl + c / 2));
                    }
                }
            }
        }
    } else if (NL > 1 && warp < 12) {
        // ---------------- epilogue 2 --------------------------------------------
        const int q = warp - 8, r = q * 32 + lane;
        const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
        uint8_t tq0 = truth_of(first, r), tq1 = truth_of(first + 1, r);  // two tiles ahead
        for (int j = 0; j < ntile; ++j) {
            const int i = ib + j;
            const int sl = i & 1;
            const uint32_t ph = (i >> 1) & 1;
            const uint8_t truth = tq0;
            tq0 = tq1;
            tq1 = truth_of(first + j + 2, r);
            wait(0, bar(kM2Done + sl), ph);
            asm volatile("tcgen05.fence::after_thread_sync;");
            uint32_t v2[H / 16][16];
            drain(kD + sl * H, trow, v2);
            ws_arrive(bar(kDEmpty + sl));
            finish(i, first + j, r, v2, bias + H, truth);
        }
    } else if (warp == R::kMma1Warp || warp == R::kMma1Warp + 1) {
        // ---------------- layer-1 issuers: even / odd tiles (elected lane) -------
        constexpr uint32_t id1 = umma_idesc_tf32(H);
        const uint64_t b1hd = umma_desc(tc_s2u(b1h), 128, KB0 * 128), b1ld = umma_desc(tc_s2u(b1l), 128, KB0 * 128);
        const int sl = warp - R::kMma1Warp;
        // two layers: accumulate into A2[sl]'s hi half, free once tile i-2's
        // layer-2 MMAs are done -- one hand-off earlier than D, which waits
        // for the final epilogue's drain (one hidden layer: D)
        const uint32_t dcol = NL > 1 ? tmem + kA2 + sl * kA2S : tmem + kD + sl * H;
        for (int i = ib + ((sl ^ ib) & 1); i < ib + ntile; i += 2) {
            const uint32_t ph = (i >> 1) & 1;
            wait(0, bar(kA1Full + sl), ph);
            wait(1, bar(NL > 1 ? kM2Done + sl : kDEmpty + sl), ph ^ 1);  // tile i-2's slot is free
            asm volatile("tcgen05.fence::after_thread_sync;");
            if (lane == 0) {
                if constexpr (kA1T) {
                    const uint32_t ah = tmem + kA1 + sl * kA1S;
#pragma unroll
                    for (int kk = 0; kk < W0 / 8; ++kk) {
                        const uint64_t ko = (uint64_t)(kk * 16);  // 256 B per k-step, in 16-byte units
                        umma_tf32_ta(dcol, ah + 8 * kk, b1hd + ko, id1, kk > 0);
                        umma_tf32_ta(dcol, ah + 8 * kk, b1ld + ko, id1, 1);
                        umma_tf32_ta(dcol, ah + W0 + 8 * kk, b1hd + ko, id1, 1);
                    }
                } else {
                    const uint64_t ahd = umma_desc(tc_s2u(a1 + sl * 2 * A1B), 128, KB0 * 128);
                    const uint64_t ald = ahd + (A1B >> 4);
#pragma unroll
                    for (int kk = 0; kk < W0 / 8; ++kk) {
                        const uint64_t ko = (uint64_t)(kk * 16);
                        umma_tf32(dcol, ahd + ko, b1hd + ko, id1, kk > 0);
                        umma_tf32(dcol, ahd + ko, b1ld + ko, id1, 1);
                        umma_tf32(dcol, ald + ko, b1hd + ko, id1, 1);
                    }
                }
                umma_commit(bar(kM1Done + sl));
            }
            __syncwarp();
        }
    } else if (NL > 1 && (warp == R::kMma2Warp || warp == R::kMma2Warp + 1)) {
        // ---------------- layer-2 issuers: even / odd tiles, A from TMEM --------
        constexpr uint32_t id2 = umma_idesc_tf32(H);
        const uint64_t b2hd = umma_desc(tc_s2u(b2h), 128, KBH * 128), b2ld = umma_desc(tc_s2u(b2l), 128, KBH * 128);
        const int sl = warp - R::kMma2Warp;
        const uint32_t a2 = tmem + kA2 + sl * kA2S, dcol = tmem + kD + sl * H;
        for (int i = ib + ((sl ^ ib) & 1); i < ib + ntile; i += 2) {
            wait(1, bar(kDEmpty + sl), ((i >> 1) & 1) ^ 1);  // the final epilogue has drained D (tile i-2)
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                // epilogue 1 has drained D[sl] and filled this column half of A2[sl]
                wait(0, bar(kA2Full + 2 * sl + half), (i >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                if (lane == 0) {
#pragma unroll
                    for (int kk = half * H / 16; kk < (half + 1) * H / 16; ++kk) {
                        const uint64_t ko = (uint64_t)(kk * 16);
                        umma_tf32_ta(dcol, a2 + 8 * kk, b2hd + ko, id2, kk > 0);
                        umma_tf32_ta(dcol, a2 + 8 * kk, b2ld + ko, id2, 1);
                        umma_tf32_ta(dcol, a2 + H + 8 * kk, b2hd + ko, id2, 1);
                    }
                    if (half) umma_commit(bar(kM2Done + sl));
                }
                __syncwarp();
            }
        }
    }
    if ((NL == 1 ? (warp >= 4 && warp < 8) : (warp >= 8 && warp < 12)) && (p.errors || p.sym_errors) &&
        p.truth) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            my_err += __shfl_xor_sync(0xffffffffu, my_err, o);
            my_ser += __shfl_xor_sync(0xffffffffu, my_ser, o);
        }
        if (lane == 0 && my_err && p.errors) atomicAdd(p.errors + net, my_err);
        if (lane == 0 && my_ser && p.sym_errors) atomicAdd(p.sym_errors + net, my_ser);
        my_err = my_ser = 0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    ib += ntile;  // (a skipped net's segment leaves the phases alone)
    }  // segments
    if (ck) {
        cv[0] = clock64() - tstart;
        for (int c = 0; c < 6; ++c) ck[c] = cv[c];
    }
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Supported shapes: widened input 32 or 64 wide, one or two hidden layers of
// 64.  Returns NOMA_ERR_UNSUPPORTED otherwise (caller uses the FFMA kernel).
int detect_tc_launch(const DetectParams &dp, cudaStream_t st) {
    if (dp.layout != NOMA_LAYOUT_WIDEN_COMPLEX) return NOMA_ERR_UNSUPPORTED;
    const NetGeom &g = dp.g;
    const int NL = g.nd - 1;
    if (NL < 1 || NL > 2) return NOMA_ERR_UNSUPPORTED;
    for (int l = 1; l <= NL; ++l)
        if (g.dims[l] != 64) return NOMA_ERR_UNSUPPORTED;
    const int W0 = g.dims[0];
    if (W0 != 32 && W0 != 64) return NOMA_ERR_UNSUPPORTED;
    DetectTcParams p;
    p.g = g;
    p.n_nets = dp.n_nets;
    p.K = dp.K;
    p.rows = dp.rows;
    p.stride = dp.stride ? dp.stride : dp.rows;
    p.tiles = (dp.rows + 63) / 64;
    p.data = dp.data;
    p.plans = dp.plans;
    p.truth = dp.truth;
    p.soft = dp.soft;
    p.codes = dp.codes;
    p.errors = dp.errors;
    p.sym_errors = dp.sym_errors;
    p.status = dp.status;
    p.clocks = nullptr;
    if (p.tiles == 0 || p.n_nets == 0) return NOMA_OK;
    // NOMA_DETECT_CLK (diagnostics): per-role cycle counters, printed after a
    // synchronising launch; the buffer lives for this call only
    long long *clk_buf = nullptr;
    const bool clk = std::getenv("NOMA_DETECT_CLK") != nullptr &&
                     cudaMallocAsync(&clk_buf, 64 * sizeof(long long), st) == cudaSuccess;
    if (clk) {
        cudaMemsetAsync(clk_buf, 0, 64 * sizeof(long long), st);
        p.clocks = clk_buf;
    }
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // one wave, one persistent CTA per SM (the smem footprint allows one),
    // each taking an equal contiguous share of all nets' tiles: a grid of
    // (SMs / nets) x nets would leave SMs idle (C3: 144 of 148) and rounding
    // up would add a second wave that doubles the kernel time
    const long long total = (long long)p.n_nets * p.tiles;
    const int ctas = total < sms ? (int)total : sms;
    auto launch = [&](auto kern, size_t smem, int threads) -> int {
        // one CTA per SM: each allocates all 512 TMEM columns
        smem = smem < 116 * 1024 ? 116 * 1024 : smem;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(ctas);
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;  // prologue beside the producer's tail
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        const bool launched = cudaLaunchKernelEx(&cfg, kern, p) == cudaSuccess && cudaGetLastError() == cudaSuccess;
        if (clk) {  // roles: loaders, epilogue 1, epilogue 2, L1 issuers (even, odd), L2 issuers (even, odd)
            long long h[48];
            cudaMemcpyAsync(h, clk_buf, sizeof h, cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            std::fprintf(stderr, "NOMA_DETECT_CLK tiles/CTA %lld:", (total + ctas - 1) / ctas);
            for (int i = 0; i < 48; ++i) std::fprintf(stderr, " %lld", h[i]);
            std::fprintf(stderr, "\n");
            cudaFreeAsync(clk_buf, st);
        }
        return launched ? NOMA_OK : NOMA_ERR_CUDA;
    };
    if (W0 == 32 && NL == 1) return launch(detect_ws_kernel<32, 64, 1>, detect_ws_smem<32, 64, 1>(), WsRoles<32, 1>::kThreads);
    if (W0 == 32 && NL == 2) return launch(detect_ws_kernel<32, 64, 2>, detect_ws_smem<32, 64, 2>(), WsRoles<32, 2>::kThreads);
    if (W0 == 64 && NL == 1) return launch(detect_ws_kernel<64, 64, 1>, detect_ws_smem<64, 64, 1>(), WsRoles<64, 1>::kThreads);
    return launch(detect_ws_kernel<64, 64, 2>, detect_ws_smem<64, 64, 2>(), WsRoles<64, 2>::kThreads);
}

}  // namespace noma_dev
