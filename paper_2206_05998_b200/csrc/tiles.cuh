// FP32 register-tile micro-kernels shared by the training and detection
// kernels, built on the sm_100a packed FP32x2 FMA (PTX fma.rn.f32x2, SASS
// FFMA2): each instruction performs two IEEE round-to-nearest FP32 FMAs.
//
// Why FFMA2 (measured on B200, profiles/r01_microbench_ffma*.txt): a scalar
// FFMA with three register operands is register-file-read limited -- an 8x4
// register outer product reaches 42.6 TFLOP/s -- while the same outer product
// in FFMA2 (one operand broadcast with the .F32 operand form, the other a
// natural float2 half of a float4 load) reaches 68.2 TFLOP/s, within 8 % of
// the 74 TFLOP/s FP32 pipe peak.  The arithmetic per element is unchanged
// (fma.rn.f32), so this is still "FP32 FFMA" training.
//
// Layout: activations live in shared memory FEATURE-MAJOR, a[feature][row],
// with row stride kSR = 132 floats (== 4 mod 32) over the 128-row batch tile;
// weights live row-major W_l[j][c] (the reference's L_l x L_{l-1}
// orientation, hybrid_nn.hpp:17) with stride sw = FP_{l-1} + 4 (== 4 mod 32).
//
// Shared-memory wavefronts (profiles/r01_microbench_lds_wavefronts.csv): an
// LDS.128 whose quarter-warps each read one bank-disjoint address costs 2
// wavefronts, one whose quarter-warps each read 8 distinct float4s costs 4.
// Every tile reads one operand quarter-uniform and the other 8-distinct with
// an 8 x 4 register tile: 32 wavefronts per 128 FMAs per thread.  NW = warps
// of the calling CTA; all loops are warp-uniform.
#pragma once

#include "common.cuh"

namespace noma_dev {

typedef unsigned long long f2_t;  // two packed FP32 lanes (lo = first)

__device__ __forceinline__ f2_t f2_bcast(float v) {
    f2_t r;
    asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(v));
    return r;
}
__device__ __forceinline__ f2_t f2_pack(float lo, float hi) {
    f2_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float2 f2_unpack(f2_t v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
// d = a * b + d, lane-wise, IEEE rn.  `volatile` pins the source order of the
// FMAs (ptxas otherwise interleaves updates of the same accumulator a few
// instructions apart and stalls on the FFMA2 latency): every tile below is
// written accumulator-major so consecutive FMAs are independent.
__device__ __forceinline__ void f2_fma(f2_t &d, f2_t a, f2_t b) {
    asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}

template <int KK>
__device__ __forceinline__ float f4c(const float4 &v) {
    return KK == 0 ? v.x : KK == 1 ? v.y : KK == 2 ? v.z : v.w;
}

// out[j][r] = relu( bias[j] + sum_k W[j][k] in[k][r] ).  J % 32 == 0,
// Kin % 4 == 0, r < 128.  Thread tile 8 j (j0 + 4 i) x 4 r (two FP32x2
// pairs); quarter-warp = j-group (W reads quarter-uniform), lane & 7 =
// r-group; warp tile 32 j x 32 r.  If yp != null (last hidden layer) the
// epilogue also forms the final-layer partials
// yp[j-block][r] = sum_{j in block} wf[j] out[j][r] (hybrid_nn.cpp:81).
template <int NW>
__device__ __forceinline__ void tile_forward(const float *__restrict__ W, int sw,
                                             const float *__restrict__ bias,
                                             const float *__restrict__ in,
                                             float *__restrict__ out, int J, int Kin, int warp,
                                             int lane, const float *__restrict__ wf = nullptr,
                                             float *__restrict__ yp = nullptr) {
    const int rg = lane & 7, jg = lane >> 3;
    const int ntile = (J >> 5) * 4;
    for (int wt = warp; wt < ntile; wt += NW) {
        const int jb = wt >> 2;
        const int j0 = jb * 32 + jg;
        const int r0 = (wt & 3) * 32 + 4 * rg;
        f2_t acc[8][2];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = f2_bcast(bias[j0 + 4 * i]);
        const float *wp = W + j0 * sw;
        const float *ip = in + r0;
#pragma unroll 1
        for (int k = 0; k < Kin; k += 4) {
            float4 w[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) w[i] = *reinterpret_cast<const float4 *>(wp + 4 * i * sw + k);
            ulonglong2 x[4];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) x[kk] = *reinterpret_cast<const ulonglong2 *>(ip + (k + kk) * kSR);
#define NOMA_FWD_K(KK)                                                                  \
    _Pragma("unroll") for (int i = 0; i < 8; ++i) {                                     \
        const f2_t wk = f2_bcast(f4c<KK>(w[i]));                                        \
        f2_fma(acc[i][0], wk, x[KK].x);                                                 \
        f2_fma(acc[i][1], wk, x[KK].y);                                                 \
    }
            NOMA_FWD_K(0) NOMA_FWD_K(1) NOMA_FWD_K(2) NOMA_FWD_K(3)
#undef NOMA_FWD_K
        }
        float y[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float2 a = f2_unpack(acc[i][0]), b = f2_unpack(acc[i][1]);
            const float v[4] = {fmaxf(a.x, 0.f), fmaxf(a.y, 0.f), fmaxf(b.x, 0.f), fmaxf(b.y, 0.f)};
            *reinterpret_cast<float4 *>(out + (j0 + 4 * i) * kSR + r0) = make_float4(v[0], v[1], v[2], v[3]);
            if (yp) {
                const float f = wf[j0 + 4 * i];
#pragma unroll
                for (int q = 0; q < 4; ++q) y[q] = fmaf(f, v[q], y[q]);
            }
        }
        if (yp) {  // warp-uniform
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                y[q] += __shfl_xor_sync(0xffffffffu, y[q], 8);
                y[q] += __shfl_xor_sync(0xffffffffu, y[q], 16);
            }
            if (jg == 0)
                *reinterpret_cast<float4 *>(yp + jb * kBatchRows + r0) = make_float4(y[0], y[1], y[2], y[3]);
        }
    }
}

// dA[c][r] = sum_j W[j][c] dz[j][r]; then in place a[c][r] = a[c][r] > 0 ? dA : 0
// (the ReLU mask of the layer below, hybrid_nn.cpp:107, :111).  C % 32 == 0.
// Thread tile 8 c (contiguous, 2 float4 of a W row; quarter-uniform) x 4 r.
template <int NW>
__device__ __forceinline__ void tile_backward_data(const float *__restrict__ W, int sw,
                                                   const float *__restrict__ dz,
                                                   float *__restrict__ a, int C, int J,
                                                   int warp, int lane) {
    const int rg = lane & 7, cg = lane >> 3;
    const int ntile = (C >> 5) * 4;
    for (int wt = warp; wt < ntile; wt += NW) {
        const int c0 = (wt >> 2) * 32 + 8 * cg;
        const int r0 = (wt & 3) * 32 + 4 * rg;
        f2_t acc[8][2];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0ull;
#pragma unroll 2
        for (int j = 0; j < J; ++j) {
            const float4 wa = *reinterpret_cast<const float4 *>(W + j * sw + c0);
            const float4 wb = *reinterpret_cast<const float4 *>(W + j * sw + c0 + 4);
            const ulonglong2 z = *reinterpret_cast<const ulonglong2 *>(dz + j * kSR + r0);
            const float wc[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const f2_t wi = f2_bcast(wc[i]);
                f2_fma(acc[i][0], wi, z.x);
                f2_fma(acc[i][1], wi, z.y);
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float *ap = a + (c0 + i) * kSR + r0;
            const float4 x = *reinterpret_cast<const float4 *>(ap);
            const float2 p = f2_unpack(acc[i][0]), q = f2_unpack(acc[i][1]);
            *reinterpret_cast<float4 *>(ap) =
                make_float4(x.x > 0.f ? p.x : 0.f, x.y > 0.f ? p.y : 0.f,
                            x.z > 0.f ? q.x : 0.f, x.w > 0.f ? q.y : 0.f);
        }
    }
}

// Partial weight gradient over a row range [r_begin, r_end):
//   gW[j][c] = sum_r dz[j][r] ain[c][r]   (hybrid_nn.cpp:109)
//   gb[j]    = sum_r dz[j][r]             (hybrid_nn.cpp:110)
// J % 32 == 0, C % 32 == 0.  Thread tile 8 j (j0 + 4 i; quarter-uniform dz
// reads) x 4 c (c0 + 8 q; 8-distinct ain reads); warp tile 32 j x 32 c.  The
// FP32x2 lanes carry the even and odd rows of the reduction, added at the end.
// Warp task = (tile, split): `splits` contiguous row ranges per tile; split s
// writes its partial to gW + s * split_stride (summed later in fixed order).
template <int NW>
__device__ __forceinline__ void tile_weight_grad(const float *__restrict__ dz,
                                                 const float *__restrict__ ain,
                                                 float *__restrict__ gW, int sw,
                                                 float *__restrict__ gb, int J, int C,
                                                 int splits, int split_stride, int warp,
                                                 int lane, bool bias = true) {
    const int cl = lane & 7, jg = lane >> 3;
    const int ncb = C >> 5;
    const int ntile = (J >> 5) * ncb;
    // shifts instead of per-task integer division (powers of two here)
    const bool pow2 = (ncb & (ncb - 1)) == 0 && (splits & (splits - 1)) == 0;
    const int ss = __ffs(splits) - 1, cs = __ffs(ncb) - 1;
    const int rows_per_split = pow2 ? kBatchRows >> ss : kBatchRows / splits;
    for (int task = warp; task < ntile * splits; task += NW) {
        const int wt = pow2 ? task >> ss : task / splits, sp = pow2 ? task & (splits - 1) : task % splits;
        const int jb = pow2 ? wt >> cs : wt / ncb, cb = pow2 ? wt & (ncb - 1) : wt % ncb;
        const int j0 = jb * 32 + jg, c0 = cb * 32 + cl;
        const int rb = sp * rows_per_split, re = rb + rows_per_split;
        f2_t acc[8][4], sb[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            sb[i] = 0ull;
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[i][q] = 0ull;
        }
        const f2_t one = f2_bcast(1.0f);
#pragma unroll 1
        for (int r = rb; r < re; r += 4) {
            ulonglong2 x[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) x[q] = *reinterpret_cast<const ulonglong2 *>(ain + (c0 + 8 * q) * kSR + r);
#pragma unroll
            for (int ih = 0; ih < 8; ih += 4) {  // dz rows in two groups: register pressure
                ulonglong2 z[4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    z[i] = *reinterpret_cast<const ulonglong2 *>(dz + (j0 + 4 * (ih + i)) * kSR + r);
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int q = 0; q < 4; ++q) f2_fma(acc[ih + i][q], z[i].x, x[q].x);
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int q = 0; q < 4; ++q) f2_fma(acc[ih + i][q], z[i].y, x[q].y);
                if (bias && cb == 0) {  // warp-uniform: bias gradient from the same loads
#pragma unroll
                    for (int i = 0; i < 4; ++i) f2_fma(sb[ih + i], z[i].x, one);
#pragma unroll
                    for (int i = 0; i < 4; ++i) f2_fma(sb[ih + i], z[i].y, one);
                }
            }
        }
        float *gWs = gW + sp * split_stride;
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float2 v = f2_unpack(acc[i][q]);
                gWs[(j0 + 4 * i) * sw + c0 + 8 * q] = v.x + v.y;
            }
        if (bias && cb == 0 && cl == 0) {
            float *gbs = gb + sp * split_stride;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float2 v = f2_unpack(sb[i]);
                gbs[j0 + 4 * i] = v.x + v.y;
            }
        }
    }
}

}  // namespace noma_dev

namespace noma_dev {

// ---------------------------------------------------------------------------
// 4 x 4 FFMA2 tiles for the 16-warp training CTA (more warps per scheduler to
// hide the FFMA2 dependency latency; 24 shared-memory wavefronts per 32
// FFMA2 per thread).  Same layouts and contracts as the 8 x 4 tiles above.

// out[j][r]: J % 16 == 0; thread tile 4 j (j0 + 4 i, quarter-uniform W reads)
// x 4 r (two FP32x2 pairs); warp tile 16 j x 32 r.  yp blocks are 16 j wide.
template <int NW>
__device__ __forceinline__ void tile_forward44(const float *__restrict__ W, int sw,
                                               const float *__restrict__ bias,
                                               const float *__restrict__ in,
                                               float *__restrict__ out, int J, int Kin, int warp,
                                               int lane, const float *__restrict__ wf = nullptr,
                                               float *__restrict__ yp = nullptr,
                                               int R = kBatchRows) {
    const int rg = lane & 7, jg = lane >> 3;
    const int nrb = R >> 5;  // 32-row blocks (R % 32 == 0): 1, 2 or 4
    const int ntile = (J >> 4) * nrb;
    const bool pow2 = (nrb & (nrb - 1)) == 0;
    const int rs = __ffs(nrb) - 1;
    for (int wt = warp; wt < ntile; wt += NW) {
        const int jb = pow2 ? wt >> rs : wt / nrb;
        const int j0 = jb * 16 + jg;
        const int r0 = (pow2 ? wt & (nrb - 1) : wt % nrb) * 32 + 4 * rg;
        f2_t acc[4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = f2_bcast(bias[j0 + 4 * i]);
        const float *wp = W + j0 * sw;
        const float *ip = in + r0;
#pragma unroll 2
        for (int k = 0; k < Kin; k += 4) {
            float4 w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) w[i] = *reinterpret_cast<const float4 *>(wp + 4 * i * sw + k);
            ulonglong2 x[4];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) x[kk] = *reinterpret_cast<const ulonglong2 *>(ip + (k + kk) * kSR);
#define NOMA_FWD44_K(KK)                                                                \
    _Pragma("unroll") for (int i = 0; i < 4; ++i) {                                     \
        const f2_t wk = f2_bcast(f4c<KK>(w[i]));                                        \
        f2_fma(acc[i][0], wk, x[KK].x);                                                 \
        f2_fma(acc[i][1], wk, x[KK].y);                                                 \
    }
            NOMA_FWD44_K(0) NOMA_FWD44_K(1) NOMA_FWD44_K(2) NOMA_FWD44_K(3)
#undef NOMA_FWD44_K
        }
        float y[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 a = f2_unpack(acc[i][0]), b = f2_unpack(acc[i][1]);
            const float v[4] = {fmaxf(a.x, 0.f), fmaxf(a.y, 0.f), fmaxf(b.x, 0.f), fmaxf(b.y, 0.f)};
            *reinterpret_cast<float4 *>(out + (j0 + 4 * i) * kSR + r0) = make_float4(v[0], v[1], v[2], v[3]);
            if (yp) {
                const float f = wf[j0 + 4 * i];
#pragma unroll
                for (int q = 0; q < 4; ++q) y[q] = fmaf(f, v[q], y[q]);
            }
        }
        if (yp) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                y[q] += __shfl_xor_sync(0xffffffffu, y[q], 8);
                y[q] += __shfl_xor_sync(0xffffffffu, y[q], 16);
            }
            if (jg == 0)
                *reinterpret_cast<float4 *>(yp + jb * kBatchRows + r0) = make_float4(y[0], y[1], y[2], y[3]);
        }
    }
}

// dA[c][r] = sum_j W[j][c] dz[j][r], masked in place; C % 16 == 0.  Thread
// tile 4 c (one float4 of a W row, quarter-uniform) x 4 r.
template <int NW>
__device__ __forceinline__ void tile_backward_data44(const float *__restrict__ W, int sw,
                                                     const float *__restrict__ dz,
                                                     float *__restrict__ a, int C, int J,
                                                     int warp, int lane, int R = kBatchRows) {
    const int rg = lane & 7, cg = lane >> 3;
    const int nrb = R >> 5;
    const int ntile = (C >> 4) * nrb;
    const bool pow2 = (nrb & (nrb - 1)) == 0;
    const int rs = __ffs(nrb) - 1;
    for (int wt = warp; wt < ntile; wt += NW) {
        const int c0 = (pow2 ? wt >> rs : wt / nrb) * 16 + 4 * cg;
        const int r0 = (pow2 ? wt & (nrb - 1) : wt % nrb) * 32 + 4 * rg;
        f2_t acc[4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0ull;
#pragma unroll 4
        for (int j = 0; j < J; ++j) {
            const float4 w = *reinterpret_cast<const float4 *>(W + j * sw + c0);
            const ulonglong2 z = *reinterpret_cast<const ulonglong2 *>(dz + j * kSR + r0);
            const float wc[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const f2_t wi = f2_bcast(wc[i]);
                f2_fma(acc[i][0], wi, z.x);
                f2_fma(acc[i][1], wi, z.y);
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            float *ap = a + (c0 + i) * kSR + r0;
            const float4 x = *reinterpret_cast<const float4 *>(ap);
            const float2 p = f2_unpack(acc[i][0]), q = f2_unpack(acc[i][1]);
            *reinterpret_cast<float4 *>(ap) =
                make_float4(x.x > 0.f ? p.x : 0.f, x.y > 0.f ? p.y : 0.f,
                            x.z > 0.f ? q.x : 0.f, x.w > 0.f ? q.y : 0.f);
        }
    }
}

// gW / gb partials over row splits; J % 32 == 0, C % 16 == 0.  Thread tile
// 4 j (j0 + 8 i; 8-distinct dz reads) x 4 c (c0 + 4 q; quarter-uniform ain
// reads); warp tile 32 j x 16 c; FP32x2 lanes carry even / odd rows.
template <int NW>
__device__ __forceinline__ void tile_weight_grad44(const float *__restrict__ dz,
                                                   const float *__restrict__ ain,
                                                   float *__restrict__ gW, int sw,
                                                   float *__restrict__ gb, int J, int C,
                                                   int splits, int split_stride, int warp,
                                                   int lane, int R = kBatchRows, bool bias = true) {
    const int jg = lane & 7, cg = lane >> 3;
    const int ncb = C >> 4;
    const int ntile = (J >> 5) * ncb;
    // task -> (tile, split) and tile -> (jb, cb) by shifts when the counts are
    // powers of two (splits is 1 or 2; ncb = C / 16), which they are for every
    // padded width here; integer division per task cost ~3 % of the kernel
    const bool pow2 = (ncb & (ncb - 1)) == 0 && (splits & (splits - 1)) == 0;
    const int ss = __ffs(splits) - 1, cs = __ffs(ncb) - 1;
    const int rows_per_split = pow2 ? R >> ss : R / splits;
    for (int task = warp; task < ntile * splits; task += NW) {
        const int wt = pow2 ? task >> ss : task / splits, sp = pow2 ? task & (splits - 1) : task % splits;
        const int jb = pow2 ? wt >> cs : wt / ncb, cb = pow2 ? wt & (ncb - 1) : wt % ncb;
        const int j0 = jb * 32 + jg, c0 = cb * 16 + cg;
        const int rb = sp * rows_per_split, re = rb + rows_per_split;
        f2_t acc[4][4], sb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            sb[i] = 0ull;
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[i][q] = 0ull;
        }
        const f2_t one = f2_bcast(1.0f);
#pragma unroll 2
        for (int r = rb; r < re; r += 4) {
            ulonglong2 z[4], x[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) z[i] = *reinterpret_cast<const ulonglong2 *>(dz + (j0 + 8 * i) * kSR + r);
#pragma unroll
            for (int q = 0; q < 4; ++q) x[q] = *reinterpret_cast<const ulonglong2 *>(ain + (c0 + 4 * q) * kSR + r);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int q = 0; q < 4; ++q) f2_fma(acc[i][q], z[i].x, x[q].x);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int q = 0; q < 4; ++q) f2_fma(acc[i][q], z[i].y, x[q].y);
            if (bias && cb == 0) {
#pragma unroll
                for (int i = 0; i < 4; ++i) f2_fma(sb[i], z[i].x, one);
#pragma unroll
                for (int i = 0; i < 4; ++i) f2_fma(sb[i], z[i].y, one);
            }
        }
        float *gWs = gW + sp * split_stride;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float2 v = f2_unpack(acc[i][q]);
                gWs[(j0 + 8 * i) * sw + c0 + 4 * q] = v.x + v.y;
            }
        if (bias && cb == 0 && cg == 0) {
            float *gbs = gb + sp * split_stride;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 v = f2_unpack(sb[i]);
                gbs[j0 + 8 * i] = v.x + v.y;
            }
        }
    }
}

}  // namespace noma_dev
