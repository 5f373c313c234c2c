// tcgen05.mma kind::tf32 issue rate on B200: one CTA per SM, one thread
// issues back-to-back M=128, K=8 MMAs of width N (A from shared memory or
// TMEM, B from shared memory; garbage data, timing only) in a compile-time
// unrolled sequence of 16, rotating over CH independent accumulators.
// Reports cycles per MMA and the implied dense TF32 TFLOP/s of the GPU.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s2u(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

template <int N, int CH, bool ATM, int IW = 1>
__global__ void rate(int iters, long long *cyc) {
    extern __shared__ __align__(1024) char sm[];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t mbars[4];
    const int tid = threadIdx.x;
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(s2u(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid < 4) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s2u(&mbars[tid])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase;
    const int w = tid >> 5;
    if (w < IW) {  // IW warps each issue iters/IW MMAs into their own accumulators
        constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint64_t ad = desc(s2u(sm), 128, 8 * 128), bd = desc(s2u(sm + 65536), 128, 8 * 128);
        long long t0 = 0;
        for (int rep = 0; rep < 2; ++rep) {
            t0 = clock64();
            for (int it = 0; it < iters / IW; it += 16) {
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const uint32_t dcol = tm + (uint32_t)(w * (256 / IW) + (j % CH) * (256 / IW / CH));
                    const uint32_t acc = (it > 0 || j >= CH) ? 1u : 0u;
                    const uint64_t ko = (uint64_t)((j & 7) * 16);
                    if ((tid & 31) == 0) {
                        if (ATM)
                            asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;}"
                                         ::"r"(dcol), "r"(tm + 256 + (j & 7) * 8), "l"(bd + ko), "r"(idesc), "r"(acc));
                        else
                            asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;}"
                                         ::"r"(dcol), "l"(ad + ko), "l"(bd + ko), "r"(idesc), "r"(acc));
                    }
                }
            }
            if ((tid & 31) == 0) {
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s2u(&mbars[w])) : "memory");
                asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(s2u(&mbars[w])), "r"(rep) : "memory");
            }
            __syncwarp();
        }
        if (tid == 0) cyc[blockIdx.x] = clock64() - t0;  // warp 0's view (all warps' MMAs share the pipe)
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, int CH, bool ATM, int IW = 1>
void run(int sms, int clk, long long *cyc) {
    const int smem = 160 * 1024, iters = 4096;
    cudaFuncSetAttribute(rate<N, CH, ATM, IW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    rate<N, CH, ATM, IW><<<sms, 128, smem>>>(iters, cyc);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("fail\n"); return; }
    long long h[256], mx = 0;
    cudaMemcpy(h, cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
    for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
    const double cpm = (double)mx / iters;
    printf("issuing warps %d chains %d A %s N=%3d: %6.1f cycles/MMA (M*N/256 = %5.1f), %5.0f TF32 TFLOP/s at %d MHz\n", IW, CH,
           ATM ? "tmem" : "smem", N, cpm, 128.0 * N / 256, 2.0 * 128 * N * 8 * sms / cpm * (clk * 1e3) / 1e12,
           clk / 1000);
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    long long *cyc;
    cudaMalloc(&cyc, sms * sizeof(long long));
    run<64, 1, false, 2>(sms, clk, cyc);
    run<64, 1, true, 2>(sms, clk, cyc);
    run<80, 1, false, 2>(sms, clk, cyc);
    run<64, 1, true, 4>(sms, clk, cyc);
    run<64, 1, false>(sms, clk, cyc);
    run<80, 1, false>(sms, clk, cyc);
    run<128, 1, false>(sms, clk, cyc);
    run<256, 1, false>(sms, clk, cyc);
    run<64, 2, false>(sms, clk, cyc);
    run<64, 4, false>(sms, clk, cyc);
    run<80, 2, false>(sms, clk, cyc);
    run<128, 2, false>(sms, clk, cyc);
    run<64, 1, true>(sms, clk, cyc);
    run<64, 2, true>(sms, clk, cyc);
    run<64, 4, true>(sms, clk, cyc);
    run<128, 1, true>(sms, clk, cyc);
    run<256, 1, true>(sms, clk, cyc);
    return 0;
}
