// FP32 FFMA register-tile micro-kernels shared by the training and detection
// kernels.  All activations live in shared memory FEATURE-MAJOR with row
// stride kSR = 132 floats (== 4 mod 32) over the 128-row batch tile; weights
// live row-major (W_l[j][c], the reference's L_l x L_{l-1} orientation) with
// stride sw = FP_{l-1} + 4 (== 4 mod 32).  With those strides every float4
// read below is bank-conflict free and each shared-memory wavefront feeds
// >= 8 warp-FFMAs.
#pragma once

#include "common.cuh"

namespace noma_dev {

template <int KK>
__device__ __forceinline__ float f4c(const float4 &v) {
    return KK == 0 ? v.x : KK == 1 ? v.y : KK == 2 ? v.z : v.w;
}

// out[j][r] = act( bias[j] + sum_k W[j][k] in[k][r] ),  j < J (mult of 16),
// k < Kin (mult of 4), r < 128.  Thread tile 4 j (strided by 4) x 8 r.
template <bool RELU>
__device__ __forceinline__ void tile_forward(const float *__restrict__ W, int sw,
                                             const float *__restrict__ bias,
                                             const float *__restrict__ in,
                                             float *__restrict__ out, int J, int Kin, int warp,
                                             int lane) {
    const int rg = lane & 7, jg = lane >> 3;
    const int ntile = (J >> 4) * 2;
    for (int wt = warp; wt < ntile; wt += kThreads / 32) {
        const int j0 = (wt >> 1) * 16 + jg;
        const int r0 = (wt & 1) * 64 + 4 * rg;
        float acc[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float b = bias[j0 + 4 * i];
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[i][q] = b;
        }
        const float *wp = W + j0 * sw;
#pragma unroll 2
        for (int k = 0; k < Kin; k += 4) {
            float4 w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) w[i] = *reinterpret_cast<const float4 *>(wp + 4 * i * sw + k);
            const float *ip = in + k * kSR + r0;
#define NOMA_FWD_K(KK)                                                                  \
    {                                                                                   \
        const float4 xa = *reinterpret_cast<const float4 *>(ip + (KK)*kSR);             \
        const float4 xb = *reinterpret_cast<const float4 *>(ip + (KK)*kSR + 32);        \
        _Pragma("unroll") for (int i = 0; i < 4; ++i) {                                 \
            const float wk = f4c<KK>(w[i]);                                             \
            acc[i][0] = fmaf(wk, xa.x, acc[i][0]);                                      \
            acc[i][1] = fmaf(wk, xa.y, acc[i][1]);                                      \
            acc[i][2] = fmaf(wk, xa.z, acc[i][2]);                                      \
            acc[i][3] = fmaf(wk, xa.w, acc[i][3]);                                      \
            acc[i][4] = fmaf(wk, xb.x, acc[i][4]);                                      \
            acc[i][5] = fmaf(wk, xb.y, acc[i][5]);                                      \
            acc[i][6] = fmaf(wk, xb.z, acc[i][6]);                                      \
            acc[i][7] = fmaf(wk, xb.w, acc[i][7]);                                      \
        }                                                                               \
    }
            NOMA_FWD_K(0) NOMA_FWD_K(1) NOMA_FWD_K(2) NOMA_FWD_K(3)
#undef NOMA_FWD_K
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            float v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = RELU ? fmaxf(acc[i][q], 0.0f) : acc[i][q];
            float *op = out + (j0 + 4 * i) * kSR + r0;
            *reinterpret_cast<float4 *>(op) = make_float4(v[0], v[1], v[2], v[3]);
            *reinterpret_cast<float4 *>(op + 32) = make_float4(v[4], v[5], v[6], v[7]);
        }
    }
}

// dA[c][r] = sum_j W[j][c] dz[j][r]; then in place a[c][r] = a[c][r] > 0 ? dA : 0
// (the ReLU mask of the layer below, hybrid_nn.cpp:107, :111).
// c < C (mult of 16), j < J (mult of 4).  Thread tile 4 c (contiguous) x 8 r.
__device__ __forceinline__ void tile_backward_data(const float *__restrict__ W, int sw,
                                                   const float *__restrict__ dz,
                                                   float *__restrict__ a, int C, int J,
                                                   int warp, int lane) {
    const int rg = lane & 7, cg = lane >> 3;
    const int ntile = (C >> 4) * 2;
    for (int wt = warp; wt < ntile; wt += kThreads / 32) {
        const int c0 = (wt >> 1) * 16 + 4 * cg;
        const int r0 = (wt & 1) * 64 + 4 * rg;
        float acc[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[i][q] = 0.0f;
#pragma unroll 4
        for (int j = 0; j < J; ++j) {
            const float4 w = *reinterpret_cast<const float4 *>(W + j * sw + c0);
            const float4 za = *reinterpret_cast<const float4 *>(dz + j * kSR + r0);
            const float4 zb = *reinterpret_cast<const float4 *>(dz + j * kSR + r0 + 32);
            const float wc[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                acc[i][0] = fmaf(wc[i], za.x, acc[i][0]);
                acc[i][1] = fmaf(wc[i], za.y, acc[i][1]);
                acc[i][2] = fmaf(wc[i], za.z, acc[i][2]);
                acc[i][3] = fmaf(wc[i], za.w, acc[i][3]);
                acc[i][4] = fmaf(wc[i], zb.x, acc[i][4]);
                acc[i][5] = fmaf(wc[i], zb.y, acc[i][5]);
                acc[i][6] = fmaf(wc[i], zb.z, acc[i][6]);
                acc[i][7] = fmaf(wc[i], zb.w, acc[i][7]);
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            float *ap = a + (c0 + i) * kSR + r0;
            const float4 xa = *reinterpret_cast<const float4 *>(ap);
            const float4 xb = *reinterpret_cast<const float4 *>(ap + 32);
            *reinterpret_cast<float4 *>(ap) =
                make_float4(xa.x > 0.f ? acc[i][0] : 0.f, xa.y > 0.f ? acc[i][1] : 0.f,
                            xa.z > 0.f ? acc[i][2] : 0.f, xa.w > 0.f ? acc[i][3] : 0.f);
            *reinterpret_cast<float4 *>(ap + 32) =
                make_float4(xb.x > 0.f ? acc[i][4] : 0.f, xb.y > 0.f ? acc[i][5] : 0.f,
                            xb.z > 0.f ? acc[i][6] : 0.f, xb.w > 0.f ? acc[i][7] : 0.f);
        }
    }
}

// gW[j][c] = sum_r dz[j][r] ain[c][r]  (hybrid_nn.cpp:109) and
// gb[j] = sum_r dz[j][r]               (hybrid_nn.cpp:110).
// j < J (mult of 32), c < C (mult of 16).  Thread tile 4 j (stride 8) x 4 c (stride 4).
__device__ __forceinline__ void tile_weight_grad(const float *__restrict__ dz,
                                                 const float *__restrict__ ain,
                                                 float *__restrict__ gW, int sw,
                                                 float *__restrict__ gb, int J, int C, int warp,
                                                 int lane) {
    const int jg = lane & 7, cg = lane >> 3;
    const int ncb = C >> 4;
    const int ntile = (J >> 5) * ncb;
    for (int wt = warp; wt < ntile; wt += kThreads / 32) {
        const int jb = wt / ncb, cb = wt % ncb;
        const int j0 = jb * 32 + jg, c0 = cb * 16 + cg;
        float acc[4][4], sb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            sb[i] = 0.f;
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[i][q] = 0.f;
        }
#pragma unroll 2
        for (int r = 0; r < kBatchRows; r += 4) {
            float4 z[4], x[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) z[i] = *reinterpret_cast<const float4 *>(dz + (j0 + 8 * i) * kSR + r);
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = *reinterpret_cast<const float4 *>(ain + (c0 + 4 * i) * kSR + r);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    float s = acc[i][q];
                    s = fmaf(z[i].x, x[q].x, s);
                    s = fmaf(z[i].y, x[q].y, s);
                    s = fmaf(z[i].z, x[q].z, s);
                    s = fmaf(z[i].w, x[q].w, s);
                    acc[i][q] = s;
                }
            if (cb == 0) {
#pragma unroll
                for (int i = 0; i < 4; ++i) sb[i] += (z[i].x + z[i].y) + (z[i].z + z[i].w);
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int q = 0; q < 4; ++q) gW[(j0 + 8 * i) * sw + c0 + 4 * q] = acc[i][q];
        if (cb == 0 && cg == 0) {
#pragma unroll
            for (int i = 0; i < 4; ++i) gb[j0 + 8 * i] = sb[i];
        }
    }
}

}  // namespace noma_dev
