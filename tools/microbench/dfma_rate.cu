// FP64 FMA throughput and latency on this part (one CTA per SM, 8 independent
// chains per thread for throughput; one chain for latency).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void tput(double *out, int iters, long long *cyc) {
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
    const double b = 0.999999, c = 1e-7;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
    long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat(double *out, int iters, long long *cyc) {
    double a = threadIdx.x * 1e-3;
    const double b = 0.999999, c = 1e-7;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) a = fma(a, b, c);
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void ffma_tput(float *out, int iters, long long *cyc) {
    float a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
    const float b = 0.999999f, c = 1e-7f;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], b, c);
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    double *o; float *of; long long *c, h;
    cudaMalloc(&o, 1 << 24); cudaMalloc(&of, 1 << 24); cudaMalloc(&c, 8);
    const int iters = 4096, thr = 512;
    tput<<<1, thr>>>(o, iters, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    tput<<<1, thr>>>(o, iters, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA per clk per SM (512 thr x 8 chains): %.2f\n", (double)thr * 8 * iters / h);
    lat<<<1, 32>>>(o, iters, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.2f clk\n", (double)h / iters);
    ffma_tput<<<1, thr>>>(of, iters, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    ffma_tput<<<1, thr>>>(of, iters, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("FFMA per clk per SM: %.2f\n", (double)thr * 8 * iters / h);
    return 0;
}
