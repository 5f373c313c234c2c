// FP32 FFMA register-tile micro-kernels shared by the training and detection
// kernels.
//
// Layout: activations live in shared memory FEATURE-MAJOR, a[feature][row],
// with row stride kSR = 132 floats (== 4 mod 32) over the 128-row batch tile;
// weights live row-major W_l[j][c] (the reference's L_l x L_{l-1}
// orientation, hybrid_nn.hpp:17) with stride sw = FP_{l-1} + 4 (== 4 mod 32).
//
// Shared-memory bandwidth is the co-bottleneck of these small GEMMs (per
// step the outputs are only J x 128).  Measured on B200 (profiles/
// r01_microbench_lds_wavefronts.csv): an LDS.128 whose four quarter-warps each
// read one (different, bank-disjoint) address costs 2 wavefronts; one whose
// quarter-warps each read 8 distinct float4s costs 4.  Every tile below is
// arranged so that one operand is quarter-uniform (2 wavefronts) and the
// other is read 8-distinct per quarter (4 wavefronts), with an 8 x 4 register
// tile: 32 wavefronts per 128 warp-FFMAs -- exactly the 4 FFMA / wavefront
// the SM sustains (4 FFMA warp-instr/clk vs 1 wavefront/clk).  NW = warps of
// the calling CTA; all loops are warp-uniform.
#pragma once

#include "common.cuh"

namespace noma_dev {

template <int KK>
__device__ __forceinline__ float f4c(const float4 &v) {
    return KK == 0 ? v.x : KK == 1 ? v.y : KK == 2 ? v.z : v.w;
}

// out[j][r] = relu( bias[j] + sum_k W[j][k] in[k][r] ).  J % 32 == 0,
// Kin % 4 == 0, r < 128.  Thread tile 8 j (j0 + 4 i) x 4 r; quarter-warp =
// j-group (W reads quarter-uniform), lane & 7 = r-group; warp tile 32 j x 32 r.
// If yp != null (last hidden layer) the epilogue also forms the final-layer
// partials yp[j-block][r] = sum_{j in block} wf[j] out[j][r] (hybrid_nn.cpp:81).
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
        float acc[8][4];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float b = bias[j0 + 4 * i];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[i][q] = b;
        }
        const float *wp = W + j0 * sw;
        const float *ip = in + r0;
#pragma unroll 1
        for (int k = 0; k < Kin; k += 4) {
            float4 w[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) w[i] = *reinterpret_cast<const float4 *>(wp + 4 * i * sw + k);
            float4 x[4];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) x[kk] = *reinterpret_cast<const float4 *>(ip + (k + kk) * kSR);
#define NOMA_FWD_K(KK)                                                                  \
    _Pragma("unroll") for (int i = 0; i < 8; ++i) {                                     \
        const float wk = f4c<KK>(w[i]);                                                 \
        acc[i][0] = fmaf(wk, x[KK].x, acc[i][0]);                                       \
        acc[i][1] = fmaf(wk, x[KK].y, acc[i][1]);                                       \
        acc[i][2] = fmaf(wk, x[KK].z, acc[i][2]);                                       \
        acc[i][3] = fmaf(wk, x[KK].w, acc[i][3]);                                       \
    }
            NOMA_FWD_K(0) NOMA_FWD_K(1) NOMA_FWD_K(2) NOMA_FWD_K(3)
#undef NOMA_FWD_K
        }
        float y[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) v[q] = fmaxf(acc[i][q], 0.0f);
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
        float acc[8][4];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[i][q] = 0.0f;
#pragma unroll 2
        for (int j = 0; j < J; ++j) {
            const float4 wa = *reinterpret_cast<const float4 *>(W + j * sw + c0);
            const float4 wb = *reinterpret_cast<const float4 *>(W + j * sw + c0 + 4);
            const float4 z = *reinterpret_cast<const float4 *>(dz + j * kSR + r0);
            const float wc[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                acc[i][0] = fmaf(wc[i], z.x, acc[i][0]);
                acc[i][1] = fmaf(wc[i], z.y, acc[i][1]);
                acc[i][2] = fmaf(wc[i], z.z, acc[i][2]);
                acc[i][3] = fmaf(wc[i], z.w, acc[i][3]);
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float *ap = a + (c0 + i) * kSR + r0;
            const float4 x = *reinterpret_cast<const float4 *>(ap);
            *reinterpret_cast<float4 *>(ap) =
                make_float4(x.x > 0.f ? acc[i][0] : 0.f, x.y > 0.f ? acc[i][1] : 0.f,
                            x.z > 0.f ? acc[i][2] : 0.f, x.w > 0.f ? acc[i][3] : 0.f);
        }
    }
}

// Partial weight gradient over a row range [r_begin, r_end):
//   gW[j][c] = sum_r dz[j][r] ain[c][r]   (hybrid_nn.cpp:109)
//   gb[j]    = sum_r dz[j][r]             (hybrid_nn.cpp:110)
// J % 32 == 0, C % 32 == 0.  Thread tile 8 j (j0 + 4 i; quarter-uniform dz
// reads) x 4 c (c0 + 8 q; 8-distinct ain reads); warp tile 32 j x 32 c.
// Warp task = (tile, split): `splits` contiguous row ranges per tile; split s
// writes its partial to gW + s * split_stride (summed later in fixed order).
template <int NW>
__device__ __forceinline__ void tile_weight_grad(const float *__restrict__ dz,
                                                 const float *__restrict__ ain,
                                                 float *__restrict__ gW, int sw,
                                                 float *__restrict__ gb, int J, int C,
                                                 int splits, int split_stride, int warp,
                                                 int lane) {
    const int cl = lane & 7, jg = lane >> 3;
    const int ncb = C >> 5;
    const int ntile = (J >> 5) * ncb;
    const int rows_per_split = kBatchRows / splits;
    for (int task = warp; task < ntile * splits; task += NW) {
        const int wt = task / splits, sp = task % splits;
        const int jb = wt / ncb, cb = wt % ncb;
        const int j0 = jb * 32 + jg, c0 = cb * 32 + cl;
        const int rb = sp * rows_per_split, re = rb + rows_per_split;
        float acc[8][4], sb[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            sb[i] = 0.f;
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[i][q] = 0.f;
        }
#pragma unroll 1
        for (int r = rb; r < re; r += 4) {
            float4 z[8], x[4];
#pragma unroll
            for (int i = 0; i < 8; ++i) z[i] = *reinterpret_cast<const float4 *>(dz + (j0 + 4 * i) * kSR + r);
#pragma unroll
            for (int q = 0; q < 4; ++q) x[q] = *reinterpret_cast<const float4 *>(ain + (c0 + 8 * q) * kSR + r);
            // component-major order: 32 independent FMAs between dependent ones
#define NOMA_GRAD_C(KK)                                                                 \
    _Pragma("unroll") for (int i = 0; i < 8; ++i) {                                     \
        const float zi = f4c<KK>(z[i]);                                                 \
        _Pragma("unroll") for (int q = 0; q < 4; ++q)                                   \
            acc[i][q] = fmaf(zi, f4c<KK>(x[q]), acc[i][q]);                             \
    }
            NOMA_GRAD_C(0) NOMA_GRAD_C(1) NOMA_GRAD_C(2) NOMA_GRAD_C(3)
#undef NOMA_GRAD_C
            if (cb == 0) {  // warp-uniform
#pragma unroll
                for (int i = 0; i < 8; ++i) sb[i] += (z[i].x + z[i].y) + (z[i].z + z[i].w);
            }
        }
        float *gWs = gW + sp * split_stride;
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int q = 0; q < 4; ++q) gWs[(j0 + 4 * i) * sw + c0 + 8 * q] = acc[i][q];
        if (cb == 0 && cl == 0) {
            float *gbs = gb + sp * split_stride;
#pragma unroll
            for (int i = 0; i < 8; ++i) gbs[j0 + 4 * i] = sb[i];
        }
    }
}

}  // namespace noma_dev
