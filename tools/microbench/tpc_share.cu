// Does an SM's FP32 throughput depend on whether the other SM of its TPC is
// busy?  Runs the same FFMA2 / FFMA / LDS-bound loops with 1, 74, 148 and 296
// CTAs (512 threads, one CTA per SM by shared-memory reservation) and reports
// the mean per-CTA cycles (clock64).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void ffma2(unsigned long long &d, unsigned long long a, unsigned long long b) {
    asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}

template <int KIND>
__global__ void k(long long *cyc, float *out, int iters) {
    extern __shared__ float sm[];
    const long long t0 = clock64();
    float s = 0.f;
    if (KIND == 0) {  // FFMA2 8x2 packed outer product
        unsigned long long acc[8][2], wp[8], xp[2];
        for (int i = 0; i < 8; ++i) {
            float w = 1e-3f * (threadIdx.x + i);
            asm("mov.b64 %0, {%1, %1};" : "=l"(wp[i]) : "f"(w));
            acc[i][0] = acc[i][1] = 0ull;
        }
        xp[0] = 0x3f0000003e800000ull;
        xp[1] = 0x3f4000003e000000ull ^ threadIdx.x;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    ffma2(acc[i][0], wp[i], xp[0]);
                    ffma2(acc[i][1], wp[i], xp[1]);
                }
        }
        for (int i = 0; i < 8; ++i) s += __int_as_float((int)(acc[i][0] ^ acc[i][1]));
    } else if (KIND == 1) {  // scalar FFMA 8x4 outer product
        float acc[8][4], w[8], v[4];
        for (int i = 0; i < 8; ++i) {
            w[i] = 1e-3f * (threadIdx.x + i);
            for (int q = 0; q < 4; ++q) acc[i][q] = 0.f;
        }
        for (int q = 0; q < 4; ++q) v[q] = 0.5f + q;
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc[i][q] = fmaf(w[i], v[q], acc[i][q]);
        for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][3];
    } else {  // LDS.128 streaming (8-distinct per quarter pattern)
        for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i;
        __syncthreads();
        float4 a = make_float4(0, 0, 0, 0);
        const int lane = threadIdx.x & 31;
        for (int it = 0; it < iters; ++it) {
            const float4 v = *reinterpret_cast<float4 *>(sm + ((it * 132 + 4 * (lane & 7)) & 4095));
            a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
        }
        s = a.x + a.y + a.z + a.w;
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (s == 1.2345f) out[0] = s;
}

int main() {
    long long *cyc;
    float *out;
    cudaMalloc(&cyc, 4096 * sizeof(long long));
    cudaMalloc(&out, 16);
    const int smem = 150 * 1024;  // forces one CTA per SM
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    long long h[4096];
    for (int kind = 0; kind < 3; ++kind)
        for (int blocks : {1, 2, 74, 148, 296}) {
            const int iters = kind == 2 ? 20000 : 2000;
            for (int rep = 0; rep < 2; ++rep) {
                if (kind == 0) k<0><<<blocks, 512, smem>>>(cyc, out, iters);
                if (kind == 1) k<1><<<blocks, 512, smem>>>(cyc, out, iters);
                if (kind == 2) k<2><<<blocks, 512, smem>>>(cyc, out, iters);
                cudaDeviceSynchronize();
            }
            cudaMemcpy(h, cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
            double m = 0;
            for (int b = 0; b < blocks; ++b) m += h[b];
            printf("%s blocks %3d: mean cycles per CTA %.0f\n",
                   kind == 0 ? "FFMA2 " : kind == 1 ? "FFMA  " : "LDS128", blocks, m / blocks);
        }
    return 0;
}
