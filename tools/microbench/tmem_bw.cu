// TMEM read / write throughput on B200: W warps per CTA (one CTA per SM),
// each repeatedly loads (tcgen05.ld.32x32b.x16 + wait::ld) or stores
// (tcgen05.st.32x32b.x16 + wait::st) 16 columns of its 32-lane quadrant.
// Reports bytes per cycle per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s2u(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <bool ST, int BATCH>
__global__ void bw(int iters, long long *cyc, unsigned *sink) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(s2u(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t t = tbase + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 128);
    unsigned acc = 0;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t r[BATCH][16];
#pragma unroll
        for (int b = 0; b < BATCH; ++b) {
            if (ST) {
#pragma unroll
                for (int i = 0; i < 16; ++i) r[b][i] = it + i;
                asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                             ::"r"(t + 16 * b), "r"(r[b][0]), "r"(r[b][1]), "r"(r[b][2]), "r"(r[b][3]), "r"(r[b][4]), "r"(r[b][5]),
                             "r"(r[b][6]), "r"(r[b][7]), "r"(r[b][8]), "r"(r[b][9]), "r"(r[b][10]), "r"(r[b][11]), "r"(r[b][12]),
                             "r"(r[b][13]), "r"(r[b][14]), "r"(r[b][15]));
            } else {
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                             : "=r"(r[b][0]), "=r"(r[b][1]), "=r"(r[b][2]), "=r"(r[b][3]), "=r"(r[b][4]), "=r"(r[b][5]), "=r"(r[b][6]),
                               "=r"(r[b][7]), "=r"(r[b][8]), "=r"(r[b][9]), "=r"(r[b][10]), "=r"(r[b][11]), "=r"(r[b][12]),
                               "=r"(r[b][13]), "=r"(r[b][14]), "=r"(r[b][15])
                             : "r"(t + 16 * b));
            }
        }
        if (ST) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        else asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int b = 0; b < BATCH; ++b) acc += r[b][0] ^ r[b][15];
    }
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
    if (acc == 0x12345) sink[0] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

template <bool ST, int BATCH>
void run(int sms, int warps, long long *cyc, unsigned *sink) {
    const int iters = 4096;
    bw<ST, BATCH><<<sms, 32 * warps>>>(iters, cyc, sink);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("fail\n"); return; }
    long long h[256], mx = 0;
    cudaMemcpy(h, cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
    for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
    const double bytes = (double)iters * BATCH * warps * 32 * 16 * 4;
    printf("%s warps %2d batch %d: %.1f B/cycle/SM\n", ST ? "st" : "ld", warps, BATCH, bytes / mx);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long *cyc;
    unsigned *sink;
    cudaMalloc(&cyc, sms * sizeof(long long));
    cudaMalloc(&sink, 4);
    for (int w : {4, 8, 16}) {
        run<false, 1>(sms, w, cyc, sink);
        run<false, 4>(sms, w, cyc, sink);
        run<true, 1>(sms, w, cyc, sink);
        run<true, 4>(sms, w, cyc, sink);
    }
    return 0;
}
