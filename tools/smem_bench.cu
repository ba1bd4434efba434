// Microbenchmark (development tool): throughput of lane-private shared-memory
// read-modify-write forms on sm_100a. Each lane owns a column of 42 int64 words
// (thread-minor layout, as in k_accumulate) and adds to pseudo-random digits.
//   mode 0: LDS.64 + IADD + STS.64  (two chunks per summand, digits i and i+1)
//   mode 1: atomicAdd (ATOMS.ADD.64) on the same addresses
//   mode 2: red.shared.add.u64 (no return value)
//   mode 3: red.shared.add.u32 x2 (32-bit halves, no carry handling: throughput only)
#include <cuda_runtime.h>
#include <stdint.h>

template <int MODE>
__global__ void __launch_bounds__(512, 1) k_smem(uint64_t* out, int iters, uint32_t seed) {
    extern __shared__ unsigned long long win[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long* col = win + warp * (42 * 32) + lane;
    for (int j = 0; j < 42; ++j) col[j * 32] = 0;
    __syncwarp();
    uint32_t x = seed ^ (threadIdx.x * 0x9E3779B9u) ^ (blockIdx.x * 0x85EBCA6Bu);
    unsigned long long acc = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            x = x * 1664525u + 1013904223u;
            uint32_t i = (x >> 16) % 40u;
            unsigned long long c0 = x, c1 = x >> 3;
            unsigned long long* p = col + i * 32;
            if (MODE == 0) {
                p[0] += c0;
                p[32] += c1;
            } else if (MODE == 1) {
                atomicAdd(p, c0);
                atomicAdd(p + 32, c1);
            } else if (MODE == 2) {
                asm volatile("red.shared.add.u64 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(p)), "l"(c0));
                asm volatile("red.shared.add.u64 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(p + 32)), "l"(c1));
            } else if (MODE == 3) {
                uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
                asm volatile("red.shared.add.u32 [%0], %1;" :: "r"(a), "r"((uint32_t)c0));
                asm volatile("red.shared.add.u32 [%0], %1;" :: "r"(a + 256), "r"((uint32_t)c1));
            } else if (MODE == 4) {          // stores only, random digit per lane
                p[0] = c0;
                p[32] = c1;
            } else if (MODE == 5) {          // loads only, random digit per lane
                acc += p[0] ^ p[32];
            } else if (MODE == 6) {          // RMW, all lanes on the same digit
                unsigned long long* q = col + ((x >> 16) & 0) * 32 + (it & 7) * 32;
                q[0] += c0;
                q[32] += c1;
            } else if (MODE == 7) {          // RMW, lanes 16-31 shifted by one digit row
                p[0] += c0;
                p[32] += c1;
            }
        }
    }
    __syncwarp();
    for (int j = 0; j < 42; ++j) acc += col[j * 32];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

extern "C" int smem_bench(int mode, uint64_t* out, int blocks, int iters, void* stream) {
    size_t smem = 16 * 42 * 32 * 8;
    cudaStream_t s = (cudaStream_t)stream;
    switch (mode) {
        case 0: cudaFuncSetAttribute(k_smem<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                k_smem<0><<<blocks, 512, smem, s>>>(out, iters, 1u); break;
        case 1: cudaFuncSetAttribute(k_smem<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                k_smem<1><<<blocks, 512, smem, s>>>(out, iters, 1u); break;
        case 2: cudaFuncSetAttribute(k_smem<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                k_smem<2><<<blocks, 512, smem, s>>>(out, iters, 1u); break;
        case 3: cudaFuncSetAttribute(k_smem<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                k_smem<3><<<blocks, 512, smem, s>>>(out, iters, 1u); break;
        case 4: cudaFuncSetAttribute(k_smem<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                k_smem<4><<<blocks, 512, smem, s>>>(out, iters, 1u); break;
        case 5: cudaFuncSetAttribute(k_smem<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                k_smem<5><<<blocks, 512, smem, s>>>(out, iters, 1u); break;
        case 6: cudaFuncSetAttribute(k_smem<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                k_smem<6><<<blocks, 512, smem, s>>>(out, iters, 1u); break;
        default: return 1;
    }
    return (int)cudaGetLastError();
}
