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
// Per CTA (128 threads, one user network, a persistent loop over 128-row
// tiles = 64 QPSK symbols of the user's slot):
//   * thread t forms widened row t of the tile (row 2s = [Re x_s; Im x_s],
//     2s+1 = [Im x_s; -Re x_s], iq_transform.cpp:17-20) straight from the
//     complex samples, splits it hi/lo and stores it in the no-swizzle
//     K-major core-matrix layout (8 rows x 16 B per core matrix);
//   * one thread issues tcgen05.mma kind::tf32 (M=128): layer 1 with
//     N = H + 16, the extra B row being the linear-branch weight w0, so the
//     TMEM accumulator column H holds x . w0; layer 2 (if any) with N = H;
//   * each thread reads its row's accumulators (tcgen05.ld 32x32b, all in
//     flight, one wait), adds the bias, applies ReLU, and either writes the
//     layer-2 A operand (hi/lo) into TMEM with tcgen05.st -- the layer-2
//     MMAs read A from TMEM -- or forms yhat = x.w0 + a_N . w_final; lane
//     pairs (2s, 2s+1) give Re/Im of symbol s, whose sign bits are the QPSK
//     decision (ties -> 0); errors against the truth codes are warp-reduced
//     into one atomic per warp.
// The next tile's samples are prefetched into registers a tile ahead and
// staged into the (then free) smem A1 buffer while layer 2 runs.
#include "kernels.cuh"

namespace noma_dev {

namespace {

constexpr int kTcGroups = 2;    // independent 128-thread tile streams per CTA
constexpr int kTcThreads = 128 * kTcGroups;
constexpr int kTcRows = 128;

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
__device__ __forceinline__ void tc_mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\nTCW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra TCW_%=;\n}" ::"r"(bar),
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
    *reinterpret_cast<float4 *>(lo + o) = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
}

}  // namespace

struct DetectTcParams {
    NetGeom g;
    int n_nets, K, rows, tiles;  // rows = data symbols per slot; tiles of 64 symbols
    const float *data;           // [S][rows][M] complex f32
    const float *plans;
    const uint8_t *truth;        // [S][rows][K] codes, nullable
    float *soft;                 // [net][rows] complex, nullable
    uint8_t *codes;              // [net][rows], nullable
    uint32_t *errors;            // [net], nullable
    const int *status;
};

// W0 = input width 2M, H = hidden width, NL = hidden layers (1 or 2).
// kTcGroups groups of 128 threads each run their own tile stream (own A1
// buffer, TMEM columns and mbarrier; group-local named barriers), so one
// group's MMAs overlap another group's epilogue; the weights are shared.
// TMEM per group (256 columns): D1 = [x W1^T | x w0] in columns 0..N1, D2
// reuses columns 0..H once D1 has been read; the layer-2 A operand a1 (hi,
// lo) is written by the epilogue into columns 128.. and 192.. with
// tcgen05.st and read from there by the layer-2 MMAs, so the group's smem A1
// buffer is free as soon as layer 1 completes and the next tile is staged
// into it while layer 2 runs.
template <int W0, int H, int NL>
constexpr uint32_t tc_abuf_bytes() {  // per group: the layer-1 A operand (hi, lo)
    return (uint32_t)(2 * kTcRows * W0 * 4);
}
template <int W0, int H, int NL>
__global__ void __launch_bounds__(kTcThreads, 1) detect_tc_kernel(DetectTcParams p) {
    constexpr int M = W0 / 2;
    constexpr int N1 = H + 16;                 // layer-1 B rows: W1 | w0 | zeros
    constexpr int KB0 = W0 / 4, KBH = H / 4;   // k-blocks per row group
    constexpr uint32_t A1B = kTcRows * W0 * 4, B1B = N1 * W0 * 4;
    constexpr uint32_t B2B = H * H * 4;
    constexpr uint32_t ABUF = tc_abuf_bytes<W0, H, NL>();
    constexpr uint32_t kA2Hi = 128, kA2Lo = 192;  // TMEM columns of the layer-2 A operand
    static_assert(N1 <= 128 && H <= 64, "TMEM column plan: D1 < 128, A2 hi/lo 64 columns each");
    extern __shared__ __align__(1024) char smem[];
    char *b1h = smem, *b1l = b1h + B1B;
    char *b2h = b1l + B1B, *b2l = b2h + (NL > 1 ? B2B : 0);
    char *abase = b2l + (NL > 1 ? B2B : 0);
    float *bias = reinterpret_cast<float *>(abase + kTcGroups * ABUF);  // [NL][H]
    float *wf = bias + NL * H;                                           // [H]
    uint64_t *mbars = reinterpret_cast<uint64_t *>(wf + H);              // [kTcGroups]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(mbars + kTcGroups);

    const int net = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = threadIdx.x >> 7, tid = threadIdx.x & 127;  // group, thread in group
    char *a1h = abase + grp * ABUF, *a1l = a1h + A1B;
    auto gsync = [&]() { asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory"); };
    if (p.status && p.status[net] != NOMA_OK) {
        if (blockIdx.x == 0 && tid == 0 && p.errors) p.errors[net] = 0xFFFFFFFFu;
        return;
    }
    const NetGeom &g = p.g;
    const int d = net / p.K, k = net % p.K;
    const float *pl = p.plans + (size_t)net * g.plan_total;

    // ---- weights: hi/lo planes in the K-major core layout (FusedPlan order) --
    for (int i = threadIdx.x; i < N1 * KB0; i += kTcThreads) {
        const int j = i / KB0, kq = (i - j * KB0) * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j < H) v = *reinterpret_cast<const float4 *>(pl + g.plan_w[1] + j * g.plan_pad[0] + kq);
        else if (j == H) v = *reinterpret_cast<const float4 *>(pl + g.plan_w0 + kq);
        put4(b1h, b1l, j, kq, KB0, v);
    }
    if constexpr (NL > 1) {
        for (int i = threadIdx.x; i < H * KBH; i += kTcThreads) {
            const int j = i / KBH, kq = (i - j * KBH) * 4;
            put4(b2h, b2l, j, kq, KBH, *reinterpret_cast<const float4 *>(pl + g.plan_w[2] + j * g.plan_pad[1] + kq));
        }
    }
    for (int i = threadIdx.x; i < NL * H; i += kTcThreads) bias[i] = pl[g.plan_b[1 + i / H] + i % H];
    for (int i = threadIdx.x; i < H; i += kTcThreads) wf[i] = pl[g.plan_f + i];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc_s2u(tmem_slot)),
                     "n"(256 * kTcGroups));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x < kTcGroups) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc_s2u(mbars + threadIdx.x)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    // group grp: TMEM columns [256 grp, 256 grp + 256); lanes = the group's rows
    const uint32_t tmem = *tmem_slot + 256 * grp;
    const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16);  // this warp's TMEM lanes
    const uint32_t bar = tc_s2u(mbars + grp);
    uint32_t phase = 0;

    // ---- tile loop: thread t = widened row t = symbol t/2, Re/Im half t&1 --
    const int sym = tid >> 1;
    const bool odd = tid & 1;
    const float2 *src = reinterpret_cast<const float2 *>(p.data) + (size_t)d * p.rows * M;
    float2 xs[M];
    uint8_t truth_next = 0;  // truth code of the tile whose samples are in xs
    auto load_tile = [&](int tile) {
        const int s = tile * 64 + sym;
        const bool ok = tile < p.tiles && s < p.rows;
        truth_next = ok && p.truth && !odd ? p.truth[((size_t)d * p.rows + s) * p.K + k] : (uint8_t)0;
#pragma unroll
        for (int m = 0; m < M; m += 2) {
            const float4 v = ok ? *reinterpret_cast<const float4 *>(src + (size_t)s * M + m)
                                : make_float4(0.f, 0.f, 0.f, 0.f);
            xs[m] = make_float2(v.x, v.y);
            xs[m + 1] = make_float2(v.z, v.w);
        }
    };
    // widened row (iq_transform.cpp:17-20) -> layer-1 A operand (hi/lo) in smem
    auto stage_a1 = [&]() {
#pragma unroll
        for (int m = 0; m < M; m += 4) {
            float4 re = make_float4(xs[m].x, xs[m + 1].x, xs[m + 2].x, xs[m + 3].x);
            float4 im = make_float4(xs[m].y, xs[m + 1].y, xs[m + 2].y, xs[m + 3].y);
            if (!odd) {
                put4(a1h, a1l, tid, m, KB0, re);
                put4(a1h, a1l, tid, M + m, KB0, im);
            } else {
                put4(a1h, a1l, tid, m, KB0, im);
                put4(a1h, a1l, tid, M + m, KB0, make_float4(-re.x, -re.y, -re.z, -re.w));
            }
        }
    };
    // sum_c relu(v_c + b_c) w_c over 16 columns into 4 partial sums
    auto dot16 = [&](const uint32_t (&v)[16], const float *b, const float *w, float (&acc)[4]) {
#pragma unroll
        for (int q = 0; q < 16; q += 4) {
            const float4 b4 = *reinterpret_cast<const float4 *>(b + q);
            const float4 w4 = *reinterpret_cast<const float4 *>(w + q);
            acc[0] = fmaf(fmaxf(__uint_as_float(v[q]) + b4.x, 0.f), w4.x, acc[0]);
            acc[1] = fmaf(fmaxf(__uint_as_float(v[q + 1]) + b4.y, 0.f), w4.y, acc[1]);
            acc[2] = fmaf(fmaxf(__uint_as_float(v[q + 2]) + b4.z, 0.f), w4.z, acc[2]);
            acc[3] = fmaf(fmaxf(__uint_as_float(v[q + 3]) + b4.w, 0.f), w4.w, acc[3]);
        }
    };
    uint32_t my_err = 0;
    const int tstride = gridDim.x * kTcGroups;
    int tile = blockIdx.x * kTcGroups + grp;
    load_tile(tile);
    stage_a1();
    uint8_t truth_a1 = truth_next;  // truth of the tile staged in A1
    load_tile(tile + tstride);
    for (; tile < p.tiles; tile += tstride) {
        const uint8_t truth_cur = truth_a1;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;");
        gsync();
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (tid == 0) {  // layer 1 (+ linear branch): D1[128 x N1] in TMEM columns 0..N1
            constexpr uint32_t id1 = umma_idesc_tf32(N1);
#pragma unroll
            for (int kk = 0; kk < W0 / 8; ++kk) {
                const uint32_t ko = kk * 256;
                const uint64_t ah = umma_desc(tc_s2u(a1h) + ko, 128, KB0 * 128);
                const uint64_t al = umma_desc(tc_s2u(a1l) + ko, 128, KB0 * 128);
                const uint64_t bh = umma_desc(tc_s2u(b1h) + ko, 128, KB0 * 128);
                const uint64_t bl = umma_desc(tc_s2u(b1l) + ko, 128, KB0 * 128);
                umma_tf32(tmem, ah, bh, id1, kk > 0);
                umma_tf32(tmem, ah, bl, id1, 1);
                umma_tf32(tmem, al, bh, id1, 1);
            }
            umma_commit(bar);
        }
        tc_mbar_wait(bar, phase);
        phase ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;");
        // D1 -> registers: all H + 16 columns in flight, one wait
        uint32_t v1[H / 16 + 1][16];
#pragma unroll
        for (int c = 0; c <= H / 16; ++c) tmem_ld16_nw(trow + 16 * c, v1[c]);
        tmem_wait_ld();
        const float lin = __uint_as_float(v1[H / 16][0]);  // column H: x . w0
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        if constexpr (NL == 1) {
            // layer 1 done: A1 is free for the next tile
            stage_a1();
            truth_a1 = truth_next;
            load_tile(tile + 2 * tstride);
#pragma unroll
            for (int c = 0; c < H / 16; ++c) dot16(v1[c], bias + 16 * c, wf + 16 * c, acc);
        } else {
            // a1 = relu(D1 + b1) -> layer-2 A operand (hi/lo) in TMEM
#pragma unroll
            for (int c = 0; c < H / 16; ++c) {
                float hi[16], lo[16];
#pragma unroll
                for (int q = 0; q < 16; q += 4) {
                    const float4 b4 = *reinterpret_cast<const float4 *>(bias + 16 * c + q);
                    const float bq[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float a = fmaxf(__uint_as_float(v1[c][q + e]) + bq[e], 0.f);
                        hi[q + e] = tf32_hi(a);
                        lo[q + e] = a - hi[q + e];
                    }
                }
                tmem_st16(trow + kA2Hi + 16 * c, hi);
                tmem_st16(trow + kA2Lo + 16 * c, lo);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;");
            gsync();
            asm volatile("tcgen05.fence::after_thread_sync;");
            if (tid == 0) {  // layer 2: D2[128 x H] in TMEM columns 0..H, A from TMEM
                constexpr uint32_t id2 = umma_idesc_tf32(H);
#pragma unroll
                for (int kk = 0; kk < H / 8; ++kk) {
                    const uint32_t ko = kk * 256;
                    const uint64_t bh = umma_desc(tc_s2u(b2h) + ko, 128, KBH * 128);
                    const uint64_t bl = umma_desc(tc_s2u(b2l) + ko, 128, KBH * 128);
                    umma_tf32_ta(tmem, tmem + kA2Hi + 8 * kk, bh, id2, kk > 0);
                    umma_tf32_ta(tmem, tmem + kA2Hi + 8 * kk, bl, id2, 1);
                    umma_tf32_ta(tmem, tmem + kA2Lo + 8 * kk, bh, id2, 1);
                }
                umma_commit(bar);
            }
            // next tile's A1 while layer 2 runs (layer 1 has completed)
            stage_a1();
            truth_a1 = truth_next;
            load_tile(tile + 2 * tstride);
            tc_mbar_wait(bar, phase);
            phase ^= 1;
            asm volatile("tcgen05.fence::after_thread_sync;");
            uint32_t v2[H / 16][16];
#pragma unroll
            for (int c = 0; c < H / 16; ++c) tmem_ld16_nw(trow + 16 * c, v2[c]);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < H / 16; ++c) dot16(v2[c], bias + H + 16 * c, wf + 16 * c, acc);
        }
        // yhat = x.w0 + a_N . w (hybrid_nn.cpp:81); Re/Im of symbol `sym`
        const float y = lin + ((acc[0] + acc[1]) + (acc[2] + acc[3]));
        const float yo = __shfl_xor_sync(0xffffffffu, y, 1);
        const int s = tile * 64 + sym;
        if (!odd && s < p.rows) {
            const uint8_t code = (uint8_t)((y < 0.f ? 1 : 0) | (yo < 0.f ? 2 : 0));  // eval.cpp:41-42
            if (p.codes) p.codes[(size_t)net * p.rows + s] = code;
            if (p.soft) *reinterpret_cast<float2 *>(p.soft + ((size_t)net * p.rows + s) * 2) = make_float2(y, yo);
            if (p.truth) my_err += __popc((unsigned)(truth_cur ^ code) & 3u);
        }
        // this tile's TMEM reads before the next tile's layer-1 MMA overwrites D
        asm volatile("tcgen05.fence::before_thread_sync;");
    }
    if (p.errors && p.truth) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) my_err += __shfl_xor_sync(0xffffffffu, my_err, o);
        if (lane == 0 && my_err) atomicAdd(p.errors + net, my_err);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_slot), "n"(256 * kTcGroups));
}

template <int W0, int H, int NL>
constexpr size_t detect_tc_smem() {
    return 2 * (size_t)(H + 16) * W0 * 4 + (NL > 1 ? 2 * (size_t)H * H * 4 : 0) +
           (size_t)kTcGroups * tc_abuf_bytes<W0, H, NL>() + (size_t)(NL + 1) * H * 4 + 8 * kTcGroups + 8;
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
    p.tiles = (dp.rows + 63) / 64;
    p.data = dp.data;
    p.plans = dp.plans;
    p.truth = dp.truth;
    p.soft = dp.soft;
    p.codes = dp.codes;
    p.errors = dp.errors;
    p.status = dp.status;
    if (p.tiles == 0 || p.n_nets == 0) return NOMA_OK;
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // one wave, one CTA per SM (the smem footprint allows one): rounding up
    // would leave a second wave of CTAs that doubles the kernel time
    int ctas = sms / p.n_nets;
    ctas = ctas < 1 ? 1 : ctas > p.tiles ? p.tiles : ctas;
    auto launch = [&](auto kern, size_t smem) -> int {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<dim3(ctas, p.n_nets), kTcThreads, smem, st>>>(p);
        return cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;
    };
    if (W0 == 32 && NL == 1) return launch(detect_tc_kernel<32, 64, 1>, detect_tc_smem<32, 64, 1>());
    if (W0 == 32 && NL == 2) return launch(detect_tc_kernel<32, 64, 2>, detect_tc_smem<32, 64, 2>());
    if (W0 == 64 && NL == 1) return launch(detect_tc_kernel<64, 64, 1>, detect_tc_smem<64, 64, 1>());
    return launch(detect_tc_kernel<64, 64, 2>, detect_tc_smem<64, 64, 2>());
}

}  // namespace noma_dev
