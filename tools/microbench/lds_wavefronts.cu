// Microbenchmark: shared-memory wavefronts per warp-wide load pattern on
// sm_100a (read with ncu metric l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld).
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float *out, int iters) {
    __shared__ __align__(16) float s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i * 0.5f;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    float4 acc = make_float4(0, 0, 0, 0);
    float a1 = 0.f;
    for (int it = 0; it < iters; ++it) {
        const int base = (it * 64) & 2047;
        if (MODE == 0) {  // LDS.128, every lane the same address (warp-uniform)
            float4 v = *reinterpret_cast<float4 *>(s + base);
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        } else if (MODE == 1) {  // LDS.128, 8 distinct consecutive float4, lane&7
            float4 v = *reinterpret_cast<float4 *>(s + base + 4 * (lane & 7));
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        } else if (MODE == 2) {  // LDS.128, 32 distinct consecutive float4
            float4 v = *reinterpret_cast<float4 *>(s + base + 4 * lane);
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        } else if (MODE == 3) {  // LDS.32, 32 distinct consecutive
            a1 += s[base + lane];
        } else if (MODE == 4) {  // LDS.32 uniform
            a1 += s[base];
        } else if (MODE == 5) {  // LDS.128, 4 distinct (lane>>3), rows stride 132
            float4 v = *reinterpret_cast<float4 *>(s + base + 132 * (lane >> 3));
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        } else if (MODE == 6) {  // LDS.64, 16 distinct consecutive float2 (lane&15)
            float2 v = *reinterpret_cast<float2 *>(s + base + 2 * (lane & 15));
            acc.x += v.x; acc.y += v.y;
        } else if (MODE == 7) {  // LDS.128, 2 distinct addresses (lane>>4)
            float4 v = *reinterpret_cast<float4 *>(s + base + 4 * (lane >> 4));
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
    }
    if (acc.x + acc.y + acc.z + acc.w + a1 == -1.f) out[0] = 1.f;
}

int main() {
    float *out;
    cudaMalloc(&out, 16);
    const int iters = 1000;
    k<0><<<1, 32>>>(out, iters);
    k<1><<<1, 32>>>(out, iters);
    k<2><<<1, 32>>>(out, iters);
    k<3><<<1, 32>>>(out, iters);
    k<4><<<1, 32>>>(out, iters);
    k<5><<<1, 32>>>(out, iters);
    k<6><<<1, 32>>>(out, iters);
    k<7><<<1, 32>>>(out, iters);
    cudaDeviceSynchronize();
    printf("done\n");
    return 0;
}
