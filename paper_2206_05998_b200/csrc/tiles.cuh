// FP32 FFMA register-tile micro-kernels shared by the training and detection
// kernels.  All activations live in shared memory FEATURE-MAJOR with row
// stride kSR = 132 floats (== 4 mod 32) over the 128-row batch tile; weights
// live row-major (W_l[j][c], the reference's L_l x L_{l-1} orientation) with
// stride sw = FP_{l-1} + 4 (== 4 mod 32).  With those strides every float4
// read below is bank-conflict free; each shared-memory wavefront feeds 8
// warp-FFMAs.  NW = warps of the calling CTA.
#pragma once

#include "common.cuh"

namespace noma_dev {

template <int KK>
__device__ __forceinline__ float f4c(const float4 &v) {
    return KK == 0 ? v.x : KK == 1 ? v.y : KK == 2 ? v.z : v.w;
}

// out[j][r] = relu( bias[j] + sum_k W[j][k] in[k][r] ),  j < J (mult of 16),
// k < Kin (mult of 4), r < 128.  Thread tile 4 j (stride 4) x 4 r; warp tile
// 16 j x 32 r.  If YP is non-null (last hidden layer) the epilogue also forms
// the final-layer partial sums yp[j-block][r] = sum_{j in block} wf[j] out[j][r]
// (hybrid_nn.cpp:81 / :94), reduced over the warp's j lanes by two shuffles.
template <int NW>
__device__ __forceinline__ void tile_forward(const float *__restrict__ W, int sw,
                                             const float *__restrict__ bias,
                                             const float *__restrict__ in,
                                             float *__restrict__ out, int J, int Kin, int warp,
                                             int lane, const float *__restrict__ wf = nullptr,
                                             float *__restrict__ yp = nullptr) {
    const int rg = lane & 7, jg = lane >> 3;
    const int ntile = (J >> 4) * 4;
    for (int wt = warp; wt < ntile; wt += NW) {
        const int jb = wt >> 2;
        const int j0 = jb * 16 + jg;
        const int r0 = (wt & 3) * 32 + 4 * rg;
        float acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float b = bias[j0 + 4 * i];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[i][q] = b;
        }
        const float *wp = W + j0 * sw;
        const float *ip = in + r0;
#pragma unroll 2
        for (int k = 0; k < Kin; k += 4) {
            float4 w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) w[i] = *reinterpret_cast<const float4 *>(wp + 4 * i * sw + k);
#define NOMA_FWD_K(KK)                                                                  \
    {                                                                                   \
        const float4 x = *reinterpret_cast<const float4 *>(ip + (k + (KK)) * kSR);      \
        _Pragma("unroll") for (int i = 0; i < 4; ++i) {                                 \
            const float wk = f4c<KK>(w[i]);                                             \
            acc[i][0] = fmaf(wk, x.x, acc[i][0]);                                       \
            acc[i][1] = fmaf(wk, x.y, acc[i][1]);                                       \
            acc[i][2] = fmaf(wk, x.z, acc[i][2]);                                       \
            acc[i][3] = fmaf(wk, x.w, acc[i][3]);                                       \
        }                                                                               \
    }
            NOMA_FWD_K(0) NOMA_FWD_K(1) NOMA_FWD_K(2) NOMA_FWD_K(3)
#undef NOMA_FWD_K
        }
        float y[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
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
// (the ReLU mask of the layer below, hybrid_nn.cpp:107, :111).
// c < C (mult of 16), j < J (mult of 4).  Thread tile 4 c (contiguous) x 4 r.
template <int NW>
__device__ __forceinline__ void tile_backward_data(const float *__restrict__ W, int sw,
                                                   const float *__restrict__ dz,
                                                   float *__restrict__ a, int C, int J,
                                                   int warp, int lane) {
    const int rg = lane & 7, cg = lane >> 3;
    const int ntile = (C >> 4) * 4;
    for (int wt = warp; wt < ntile; wt += NW) {
        const int c0 = (wt >> 2) * 16 + 4 * cg;
        const int r0 = (wt & 3) * 32 + 4 * rg;
        float acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[i][q] = 0.0f;
#pragma unroll 4
        for (int j = 0; j < J; ++j) {
            const float4 w = *reinterpret_cast<const float4 *>(W + j * sw + c0);
            const float4 z = *reinterpret_cast<const float4 *>(dz + j * kSR + r0);
            const float wc[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                acc[i][0] = fmaf(wc[i], z.x, acc[i][0]);
                acc[i][1] = fmaf(wc[i], z.y, acc[i][1]);
                acc[i][2] = fmaf(wc[i], z.z, acc[i][2]);
                acc[i][3] = fmaf(wc[i], z.w, acc[i][3]);
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            float *ap = a + (c0 + i) * kSR + r0;
            const float4 x = *reinterpret_cast<const float4 *>(ap);
            *reinterpret_cast<float4 *>(ap) =
                make_float4(x.x > 0.f ? acc[i][0] : 0.f, x.y > 0.f ? acc[i][1] : 0.f,
                            x.z > 0.f ? acc[i][2] : 0.f, x.w > 0.f ? acc[i][3] : 0.f);
        }
    }
}

// gW[j][c] = sum_r dz[j][r] ain[c][r]  (hybrid_nn.cpp:109) and
// gb[j] = sum_r dz[j][r]               (hybrid_nn.cpp:110).
// j < J (mult of 32), c < C (mult of 8).  Thread tile 4 j (stride 8) x 2 c
// (stride 4); warp tile 32 j x 8 c.
template <int NW>
__device__ __forceinline__ void tile_weight_grad(const float *__restrict__ dz,
                                                 const float *__restrict__ ain,
                                                 float *__restrict__ gW, int sw,
                                                 float *__restrict__ gb, int J, int C, int warp,
                                                 int lane) {
    const int jg = lane & 7, cg = lane >> 3;
    const int ncb = C >> 3;
    const int ntile = (J >> 5) * ncb;
    for (int wt = warp; wt < ntile; wt += NW) {
        const int jb = wt / ncb, cb = wt % ncb;
        const int j0 = jb * 32 + jg, c0 = cb * 8 + cg;
        float acc[4][2], sb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            sb[i] = 0.f;
            acc[i][0] = acc[i][1] = 0.f;
        }
#pragma unroll 4
        for (int r = 0; r < kBatchRows; r += 4) {
            float4 z[4], x[2];
#pragma unroll
            for (int i = 0; i < 4; ++i) z[i] = *reinterpret_cast<const float4 *>(dz + (j0 + 8 * i) * kSR + r);
#pragma unroll
            for (int q = 0; q < 2; ++q) x[q] = *reinterpret_cast<const float4 *>(ain + (c0 + 4 * q) * kSR + r);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int q = 0; q < 2; ++q) {
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
            for (int q = 0; q < 2; ++q) gW[(j0 + 8 * i) * sw + c0 + 4 * q] = acc[i][q];
        if (cb == 0 && cg == 0) {
#pragma unroll
            for (int i = 0; i < 4; ++i) gb[j0 + 8 * i] = sb[i];
        }
    }
}

}  // namespace noma_dev
