// Read-bandwidth probes (bench infrastructure; no method arithmetic): how fast can one
// B200 stream a read-only array with a given load pattern and occupancy? Each thread XORs
// the 32-bit words it loads and writes one word, so the kernels are purely memory-bound.
// Used for the secondary roofline denominator ("read probe") and to separate memory-side
// limits from the accumulate kernel's on-chip limits.
#include <cuda_runtime.h>
#include <stdint.h>

template <int L2HINT>
__device__ __forceinline__ uint4 pld(const uint4* p) {
    uint4 v;
    if (L2HINT == 1)
        asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    else if (L2HINT == 2)
        asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    else
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

// tile-strided (the accumulate kernel's pattern): tile = T*U vectors, block b takes tiles b, b+G, ...
template <int U, int L2HINT>
__global__ void k_probe_tiles(const uint4* __restrict__ x, uint64_t nvec, uint32_t* out) {
    const int T = blockDim.x;
    const uint64_t TV = (uint64_t)T * U;
    const uint64_t ntiles = nvec / TV;
    uint32_t acc = 0;
    uint4 buf[U];
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
#pragma unroll
        for (int u = 0; u < U; ++u) buf[u] = pld<L2HINT>(x + t * TV + (uint64_t)u * T + threadIdx.x);
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= buf[u].x ^ buf[u].y ^ buf[u].z ^ buf[u].w;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// contiguous chunk per block (each block streams its own contiguous range)
template <int U>
__global__ void k_probe_chunks(const uint4* __restrict__ x, uint64_t nvec, uint32_t* out) {
    const uint64_t per = (nvec + gridDim.x - 1) / gridDim.x;
    const uint64_t a = blockIdx.x * per, b = min(nvec, a + per);
    uint32_t acc = 0;
    uint4 buf[U];
    const uint64_t step = (uint64_t)blockDim.x * U;
    uint64_t v = a + threadIdx.x;
    for (; v + (U - 1) * blockDim.x < b; v += step) {
#pragma unroll
        for (int u = 0; u < U; ++u) buf[u] = pld<1>(x + v + (uint64_t)u * blockDim.x);
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= buf[u].x ^ buf[u].y ^ buf[u].z ^ buf[u].w;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

extern "C" int synth_probe_read(const void* x, uint64_t nbytes, void* out, int variant, int blocks, int threads,
                                void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const uint4* v = (const uint4*)x;
    uint64_t nvec = nbytes / 16;
    uint32_t* o = (uint32_t*)out;
    switch (variant) {
        case 0: k_probe_tiles<4, 1><<<blocks, threads, 0, s>>>(v, nvec, o); break;
        case 1: k_probe_tiles<8, 1><<<blocks, threads, 0, s>>>(v, nvec, o); break;
        case 2: k_probe_tiles<4, 0><<<blocks, threads, 0, s>>>(v, nvec, o); break;
        case 3: k_probe_tiles<4, 2><<<blocks, threads, 0, s>>>(v, nvec, o); break;
        case 4: k_probe_chunks<4><<<blocks, threads, 0, s>>>(v, nvec, o); break;
        case 5: k_probe_chunks<8><<<blocks, threads, 0, s>>>(v, nvec, o); break;
        case 6: k_probe_tiles<16, 1><<<blocks, threads, 0, s>>>(v, nvec, o); break;
        default: return 1;
    }
    return (int)cudaGetLastError();
}
