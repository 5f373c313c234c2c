// Microbenchmark: FP32 FFMA throughput on sm_100a for (a) constant operands,
// (b) all-register operands in independent chains, (c) an 8x4 register
// outer product (the train/detect tile inner loop without memory).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ffma_const(float *out, int iters, float a, float b) {
    float x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
    float s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1.2345f) out[0] = s;
}

__global__ void ffma_reg(float *out, int iters) {
    float x[8], y[8], z[8];
    for (int i = 0; i < 8; ++i) {
        x[i] = threadIdx.x * 1e-3f + i;
        y[i] = 0.999f - threadIdx.x * 1e-7f * i;
        z[i] = 1e-4f * (i + 1) + threadIdx.x * 1e-9f;
    }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], y[i], z[i]);
    float s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1.2345f) out[0] = s;
}

__global__ void ffma_outer(float *out, int iters) {
    float acc[8][4], w[8], v[4];
    for (int i = 0; i < 8; ++i) {
        w[i] = 1e-3f * (threadIdx.x + i);
        for (int q = 0; q < 4; ++q) acc[i][q] = 0.f;
    }
    for (int q = 0; q < 4; ++q) v[q] = 0.5f + 1e-4f * (threadIdx.x + q);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[i][q] = fmaf(w[i], v[q], acc[i][q]);
        w[it & 7] += 1e-7f;  // keep operands live/varying
    }
    float s = 0;
    for (int i = 0; i < 8; ++i)
        for (int q = 0; q < 4; ++q) s += acc[i][q];
    if (s == 1.2345f) out[0] = s;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out;
    cudaMalloc(&out, 16);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4096;
    for (int threads : {256, 512, 1024}) {
        const int blocks = sms * (2048 / threads);
        for (int kind = 0; kind < 3; ++kind) {
            float best = 1e30f;
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(a);
                if (kind == 0) ffma_const<<<blocks, threads>>>(out, iters, 0.9999f, 1e-4f);
                if (kind == 1) ffma_reg<<<blocks, threads>>>(out, iters);
                if (kind == 2) ffma_outer<<<blocks, threads>>>(out, iters);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            const double fma_per_thread = kind == 2 ? 4.0 * 32 * iters : 16.0 * 8 * iters;
            const double tf = 2.0 * fma_per_thread * blocks * threads / (best * 1e-3) / 1e12;
            printf("threads/CTA %4d kind %s: %.1f TFLOP/s\n", threads,
                   kind == 0 ? "const-operand" : kind == 1 ? "register     " : "outer8x4     ", tf);
        }
    }
    return 0;
}
