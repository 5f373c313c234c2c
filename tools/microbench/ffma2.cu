// Microbenchmark: packed FP32x2 FMA (PTX fma.rn.f32x2 -> SASS FFMA2, sm_100a)
// vs scalar FFMA, register operands, and an 8x4 outer product built from FFMA2.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pk(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void ffma2(unsigned long long &d, unsigned long long a, unsigned long long b) {
    asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}

__global__ void reg_ffma2(float *out, int iters) {
    unsigned long long x[8], y[8], z[8];
    for (int i = 0; i < 8; ++i) {
        x[i] = pk(threadIdx.x * 1e-3f + i, 0.5f + i);
        y[i] = pk(0.999f - threadIdx.x * 1e-7f * i, 0.998f);
        z[i] = pk(1e-4f * (i + 1), 2e-4f);
    }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(y[i]), "l"(z[i]));
    unsigned long long s = 0;
    for (int i = 0; i < 8; ++i) s ^= x[i];
    if (s == 12345) out[0] = 1.f;
}

// acc[i][q-pair] += (w_i, w_i) * (x_q, x_q+1): 8 x 2 packed accumulators
__global__ void outer_ffma2(float *out, int iters) {
    unsigned long long acc[8][2], wp[8], xp[2];
    for (int i = 0; i < 8; ++i) {
        const float w = 1e-3f * (threadIdx.x + i);
        wp[i] = pk(w, w);
        acc[i][0] = acc[i][1] = 0ull;
    }
    xp[0] = pk(0.5f, 0.25f);
    xp[1] = pk(0.125f + threadIdx.x * 1e-6f, 0.75f);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                ffma2(acc[i][0], wp[i], xp[0]);
                ffma2(acc[i][1], wp[i], xp[1]);
            }
        wp[it & 7] ^= 1ull;
    }
    unsigned long long s = 0;
    for (int i = 0; i < 8; ++i) s ^= acc[i][0] ^ acc[i][1];
    if (s == 12345) out[0] = 1.f;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out;
    cudaMalloc(&out, 16);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4096, threads = 256, blocks = sms * 8;
    for (int kind = 0; kind < 2; ++kind) {
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            if (kind == 0) reg_ffma2<<<blocks, threads>>>(out, iters);
            else outer_ffma2<<<blocks, threads>>>(out, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        // kind 0: 16*8 FFMA2 per iter = 256 FMAs; kind 1: 4*8*2 FFMA2 = 128 FMAs
        const double fma = (kind == 0 ? 256.0 : 128.0) * iters * blocks * threads;
        printf("%s: %.1f TFLOP/s\n", kind == 0 ? "FFMA2 register chains " : "FFMA2 8x4 outer product", 2 * fma / (best * 1e-3) / 1e12);
    }
    return 0;
}
