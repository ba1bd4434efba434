// Microbenchmark (development tool): issue throughput of single integer SASS ops on sm_100a.
// 8 independent dependency chains per thread, 64 warps per SM; reports warp-instructions
// per clock per SM for each op (4.0 = one per SMSP per clock).
#include <cuda_runtime.h>
#include <stdint.h>

#define CHAINS 8

template <int OP>
__global__ void __launch_bounds__(1024, 2) k_op(uint32_t* out, int iters, uint32_t seed) {
    uint32_t v[CHAINS], w[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) { v[c] = seed * (threadIdx.x + c + 1); w[c] = seed ^ c; }
    const uint32_t K = seed | 1u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
            uint32_t x = v[c], r;
            if (OP == 0) asm volatile("add.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(K));                   // IADD3
            if (OP == 1) asm volatile("xor.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(K));                   // LOP3
            if (OP == 2) asm volatile("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(w[c]), "r"(K)); // SHF
            if (OP == 3) asm volatile("mad.lo.u32 %0, %1, %2, %1;" : "=r"(r) : "r"(x), "r"(K));            // IMAD
            if (OP == 4) asm volatile("mad.hi.u32 %0, %1, %2, %1;" : "=r"(r) : "r"(x), "r"(K));            // IMAD.HI
            if (OP == 5) { uint64_t t; asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(t) : "r"(x), "r"(K), "l"((uint64_t)w[c])); r = (uint32_t)t ^ (uint32_t)(t >> 32); }
            if (OP == 6) asm volatile("max.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(K));                   // VIMNMX
            if (OP == 7) asm volatile("{.reg .pred p; setp.lt.u32 p, %1, %2; selp.b32 %0, %1, %2, p;}" : "=r"(r) : "r"(x), "r"(K));
            v[c] = r;
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc ^= v[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

extern "C" int op_bench(int op, uint32_t* out, int blocks, int iters, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    switch (op) {
        case 0: k_op<0><<<blocks, 1024, 0, s>>>(out, iters, 3u); break;
        case 1: k_op<1><<<blocks, 1024, 0, s>>>(out, iters, 3u); break;
        case 2: k_op<2><<<blocks, 1024, 0, s>>>(out, iters, 3u); break;
        case 3: k_op<3><<<blocks, 1024, 0, s>>>(out, iters, 3u); break;
        case 4: k_op<4><<<blocks, 1024, 0, s>>>(out, iters, 3u); break;
        case 5: k_op<5><<<blocks, 1024, 0, s>>>(out, iters, 3u); break;
        case 6: k_op<6><<<blocks, 1024, 0, s>>>(out, iters, 3u); break;
        case 7: k_op<7><<<blocks, 1024, 0, s>>>(out, iters, 3u); break;
        default: return 1;
    }
    return (int)cudaGetLastError();
}
