// Single-CTA tcgen05.mma kind::tf32 check (M=128, N=64, K=32): validates the
// no-swizzle K-major shared-memory descriptor layout used by k_detect_tc.cu
// against a CPU reference.  Core matrix = 8 rows x 16 bytes (4 tf32) stored
// contiguously (128 B); core matrices adjacent along K are LBO bytes apart,
// along M/N SBO bytes apart.  argv[1] = 1 swaps the roles (diagnostic).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

constexpr int M = 128, N = 64, K = 32;

__device__ __forceinline__ uint32_t s2u(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version (sm100)
    // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0) at bits 61-63
    return d;
}

__global__ void k(const float *A, const float *B, float *D, int swap, uint32_t idesc_override) {
    __shared__ __align__(1024) float sa[M * K];
    __shared__ __align__(1024) float sb[N * K];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t mbar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // pack: element (r, k) -> core (r/8, k/4) at ((r/8)*(K/4) + k/4)*128 B + (r%8)*16 + (k%4)*4
    for (int i = tid; i < M * K; i += blockDim.x) {
        const int r = i / K, c = i % K;
        sa[(((r >> 3) * (K / 4) + (c >> 2)) * 128 + (r & 7) * 16 + (c & 3) * 4) / 4] = A[i];
    }
    for (int i = tid; i < N * K; i += blockDim.x) {
        const int r = i / K, c = i % K;
        sb[(((r >> 3) * (K / 4) + (c >> 2)) * 128 + (r & 7) * 16 + (c & 3) * 4) / 4] = B[i];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(s2u(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s2u(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;
    // instruction descriptor: D f32, A/B tf32, K-major both, N>>3, M>>4
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    if (idesc_override) idesc = idesc_override;
    const uint32_t lbo = swap ? (K / 4) * 128 : 128;   // K-direction core stride
    const uint32_t sbo = swap ? 128 : (K / 4) * 128;   // M/N-direction core stride
    if (tid == 0) {
        for (int kk = 0; kk < K / 8; ++kk) {
            const uint64_t ad = make_desc(s2u(sa) + kk * 2 * 128, lbo, sbo);
            const uint64_t bd = make_desc(s2u(sb) + kk * 2 * 128, lbo, sbo);
            const uint32_t acc = kk > 0;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s2u(&mbar)));
    }
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(s2u(&mbar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    // each warp reads its 32 lanes (rows) x 64 columns
    for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t v[16];
        const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int i = 0; i < 16; ++i) D[(warp * 32 + lane) * N + c0 + i] = __uint_as_float(v[i]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

int main(int argc, char **argv) {
    const int swap = argc > 1 ? atoi(argv[1]) : 0;
    float *hA = new float[M * K], *hB = new float[N * K], *hD = new float[M * N];
    srand(1);
    for (int i = 0; i < M * K; ++i) hA[i] = (rand() % 2001 - 1000) / 1000.0f;
    for (int i = 0; i < N * K; ++i) hB[i] = (rand() % 2001 - 1000) / 1000.0f;
    float *dA, *dB, *dD;
    cudaMalloc(&dA, M * K * 4);
    cudaMalloc(&dB, N * K * 4);
    cudaMalloc(&dD, M * N * 4);
    cudaMemcpy(dA, hA, M * K * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, N * K * 4, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, M * N * 4);
    k<<<1, 128>>>(dA, dB, dD, swap, 0);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    int bad = 0;
    for (int r = 0; r < M; ++r)
        for (int c = 0; c < N; ++c) {
            double ref = 0;
            for (int kk = 0; kk < K; ++kk) ref += (double)hA[r * K + kk] * hB[c * K + kk];
            const double err = fabs(ref - hD[r * N + c]);
            maxerr = fmax(maxerr, err);
            maxref = fmax(maxref, fabs(ref));
            if (err > 1e-2 && bad < 5) {
                printf("mismatch r=%d c=%d ref=%f got=%f\n", r, c, ref, hD[r * N + c]);
                ++bad;
            }
        }
    printf("swap=%d max abs err %.3e (max |ref| %.3f) -> %s\n", swap, maxerr, maxref, maxerr < 1e-2 ? "PASS" : "FAIL");
    return 0;
}
