// Minimal repro for compute-sanitizer racecheck: a producer warp writes shared
// memory (one word per lane), __syncwarp(), lane 0 arrives on an mbarrier
// (release); a consumer warp waits on it (acquire) and reads the words.
// Per-warp arrivals after __syncwarp are the hand-off used by the tcgen05
// detection pipeline.  argv[1] = 1: every lane arrives (count 32) instead.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s2u(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(int per_lane, int iters, int *bad) {
    __shared__ float buf[2][32];
    __shared__ __align__(8) uint64_t full[2], empty[2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s2u(&full[i])), "r"(per_lane ? 32 : 1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s2u(&empty[i])), "r"(per_lane ? 32 : 1));
        }
    }
    __syncthreads();
    auto arrive = [&](uint64_t *b) {
        if (per_lane) {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s2u(b)) : "memory");
        } else {
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s2u(b)) : "memory");
        }
    };
    auto wait = [&](uint64_t *b, uint32_t ph) {
        asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(s2u(b)), "r"(ph) : "memory");
    };
    for (int i = 0; i < iters; ++i) {
        const int sl = i & 1;
        const uint32_t ph = (i >> 1) & 1;
        if (warp == 0) {  // producer
            wait(&empty[sl], ph ^ 1);
            buf[sl][lane] = (float)(i * 32 + lane);
            arrive(&full[sl]);
        } else {          // consumer
            wait(&full[sl], ph);
            if (buf[sl][lane] != (float)(i * 32 + lane)) atomicAdd(bad, 1);
            arrive(&empty[sl]);
        }
    }
}

int main(int argc, char **argv) {
    int *bad;
    cudaMalloc(&bad, 4);
    cudaMemset(bad, 0, 4);
    k<<<1, 64>>>(argc > 1 ? atoi(argv[1]) : 0, 64, bad);
    cudaError_t e = cudaDeviceSynchronize();
    int h = -1;
    cudaMemcpy(&h, bad, 4, cudaMemcpyDeviceToHost);
    printf("%s (%s, bad=%d)\n", e == cudaSuccess && h == 0 ? "OK" : "BAD", cudaGetErrorString(e), h);
    return 0;
}
