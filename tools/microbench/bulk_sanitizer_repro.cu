// Minimal repro for compute-sanitizer's handling of the latency kernel's
// async-proxy copies: (1) cp.async.bulk shared::cta -> peer CTA shared::cluster
// completing on the peer's mbarrier (the a_l all-gather), (2) cp.async.bulk
// global -> shared double-buffered tiles read after an mbarrier wait (the
// per-step minibatch tile).  Both patterns are correct by the PTX memory
// model; the program checks the data it receives and prints OK / BAD.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s2u(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
    uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o;
}
__device__ __forceinline__ uint32_t rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void csync() {
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void arm(uint32_t b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void wait(uint32_t b, uint32_t ph) {
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(b), "r"(ph) : "memory");
}

constexpr int kBytes = 2112, kF = kBytes / 4, kSteps = 8;

__global__ void repro(const float *g, int *bad, int issuer, int pad, int bug, int sta, int early, int nbar) {
    extern __shared__ __align__(128) unsigned char smem[];
    float *src = (float *)(smem + pad);       // own tile
    uint32_t ncl;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(ncl));
    const uint32_t ngat = sta == 2 ? ncl : 2;  // tiles gathered per CTA
    float *dst = src + kF;                    // [ngat][kF] gathered tiles
    float *tile = dst + ngat * kF;            // [2][kF] global tiles
    uint64_t *bars = (uint64_t *)(tile + 2 * kF);  // [0] gather, [1..2] tile
    const uint32_t r = sta == 2 ? rank() : rank() & 1, pair = sta == 2 ? 0 : rank() & ~1u, tid = threadIdx.x;
    if (tid == 0) {
        for (int i = 0; i < nbar; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s2u(bars + i)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (!early) csync();
    if (tid == 0) arm(s2u(bars), ngat * kBytes);
    if (early) __syncthreads();  // init + first arm visible to the tile issuer
    if (tid == (uint32_t)issuer) {  // first tile: same issuer as the prefetches
        if (early == 2) {  // late first tile: peers' st.async land while this CTA waits on it
            const long long t0 = clock64();
            while (clock64() - t0 < 200000) {}
        }
        arm(s2u(bars + 1), kBytes);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(s2u(tile)), "l"(g), "r"(kBytes), "r"(s2u(bars + 1)) : "memory");
    }
    if (early) csync();  // the training kernel's order: first tile issued before the cluster barrier
    for (int i = tid; i < kF; i += blockDim.x) src[i] = (float)(r * 100000 + i);
    __syncthreads();
    if (sta) {  // gather by st.async.v4 (per thread) instead of one bulk copy per peer
        for (uint32_t q = 0; q < ngat; ++q)
            for (int i = 4 * tid; i < kF; i += 4 * blockDim.x) {
                const float4 v = *reinterpret_cast<const float4 *>(src + i);
                asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];"
                             ::"r"(mapa(s2u(dst + r * kF + i), pair + q)), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w),
                             "r"(mapa(s2u(bars), pair + q)) : "memory");
            }
    } else if (tid < 2) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(mapa(s2u(dst + r * kF), pair + tid)), "r"(s2u(src)), "r"(kBytes), "r"(mapa(s2u(bars), pair + tid)) : "memory");
    }
    if (early == 2) wait(s2u(bars + 1), 0);  // tile first, as the training kernel's step 0
    wait(s2u(bars), 0);
    for (int i = tid; i < (int)ngat * kF; i += blockDim.x)
        if (dst[i] != (float)((i / kF) * 100000 + i % kF)) atomicAdd(bad, 1);
    float acc = 0.f;
    for (int s = 0; s < kSteps; ++s) {
        const int b = s & 1;
        wait(s2u(bars + 1 + b), (s >> 1) & 1);
        if (tid == (uint32_t)issuer && s + 1 < kSteps) {   // prefetch next step's tile into the other buffer
            arm(s2u(bars + 1 + (b ^ 1)), kBytes);
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(s2u(tile + (b ^ 1) * kF)), "l"(g + (s + 1) * kF), "r"(kBytes), "r"(s2u(bars + 1 + (b ^ 1))) : "memory");
        }
        for (int i = tid; i < kF; i += blockDim.x) {
            if (tile[b * kF + i] != (float)(s * kF + i)) atomicAdd(bad, 1);
            acc += tile[b * kF + i];
        }
        __syncthreads();  // every read of tile[b] before the refill two steps on
    }
    if (acc == -1.f) atomicAdd(bad, 1000);
    if (bug && tid == 0) {  // deliberate: test an uninitialised barrier (shows the tool's address encoding)
        uint32_t ok;
        asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(s2u(bars + 3)) : "memory");
        if (ok == 7) atomicAdd(bad, 1);
    }
    csync();
}

int main(int argc, char **argv) {
    float *g; int *bad;
    cudaMalloc(&g, kSteps * kBytes);
    cudaMalloc(&bad, 4);
    float h[kSteps * kF];
    for (int i = 0; i < kSteps * kF; ++i) h[i] = (float)i;
    cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice);
    cudaMemset(bad, 0, 4);
    // argv[1]: thread issuing the tile copies; argv[2]: cluster size; argv[3]:
    // extra shared bytes in front (barriers at a high offset); argv[4]: threads
    const int issuer = argc > 1 ? atoi(argv[1]) : 0, cs = argc > 2 ? atoi(argv[2]) : 2;
    const int pad = argc > 3 ? atoi(argv[3]) : 0, nt = argc > 4 ? atoi(argv[4]) : 128;
    const int bug = argc > 5 ? atoi(argv[5]) : 0, sta = argc > 6 ? atoi(argv[6]) : 0,
              early = argc > 7 ? atoi(argv[7]) : 0, nbar = argc > 8 ? atoi(argv[8]) : 3;
    const int smem = (3 + (sta == 2 ? cs : 2)) * kBytes + 8 * (nbar + 1) + pad;  // bars at the end
    cudaFuncSetAttribute(repro, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(repro, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, repro, (const float *)g, bad, issuer, pad, bug, sta, early, nbar);
    cudaError_t e = cudaDeviceSynchronize();
    int hb = -1;
    cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
    printf("%s (%s, bad=%d)\n", (e == cudaSuccess && hb == 0) ? "OK" : "BAD", cudaGetErrorString(e), hb);
    return 0;
}
