// Read-bandwidth probe of the segment access pattern (development tool, standalone):
// 2^28 doubles; (a) grid-stride 16-B loads, (b) one warp per contiguous segment of L doubles
// (the k_segments_uniform pattern), for several loads-in-flight depths. Sink xor to global.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o seg_read_probe seg_read_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ld(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

template <int DEPTH>
__global__ void __launch_bounds__(256, 2) k_grid(const uint4* x, uint64_t nv, unsigned* sink) {
    unsigned acc = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (DEPTH - 1) * stride < nv; i += DEPTH * stride) {
        uint4 v[DEPTH];
#pragma unroll
        for (int d = 0; d < DEPTH; ++d) v[d] = ld(x + i + d * stride);
#pragma unroll
        for (int d = 0; d < DEPTH; ++d) acc ^= v[d].x ^ v[d].y ^ v[d].z ^ v[d].w;
    }
    for (; i < nv; i += stride) { uint4 v = ld(x + i); acc ^= v.x ^ v.y ^ v.z ^ v.w; }
    if (acc == 0x12345678u) sink[0] = acc;
}

// one warp per segment of seg_vecs 16-B vectors; DEPTH vectors per lane in flight
template <int DEPTH>
__global__ void __launch_bounds__(256, 2) k_seg(const uint4* x, uint64_t nseg, uint64_t seg_vecs, unsigned* sink) {
    const int lane = threadIdx.x & 31;
    const uint64_t nw = (uint64_t)gridDim.x * 8, gw = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    unsigned acc = 0;
    for (uint64_t s = gw; s < nseg; s += nw) {
        const uint4* p = x + s * seg_vecs + lane;
        for (uint64_t j = 0; j < seg_vecs; j += 32 * DEPTH) {
            uint4 v[DEPTH];
#pragma unroll
            for (int d = 0; d < DEPTH; ++d) v[d] = ld(p + j + d * 32);
#pragma unroll
            for (int d = 0; d < DEPTH; ++d) acc ^= v[d].x ^ v[d].y ^ v[d].z ^ v[d].w;
        }
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

// LPS lanes per segment (16: K6h's half warps, 8: quarters), 32/LPS segments per warp at a time
template <int DEPTH, int LPS>
__global__ void __launch_bounds__(256, 2) k_seg_part(const uint4* x, uint64_t nseg, uint64_t seg_vecs, unsigned* sink) {
    const int lane = threadIdx.x & 31, sl = lane % LPS, grp = lane / LPS;
    constexpr int G = 32 / LPS;
    const uint64_t nw = (uint64_t)gridDim.x * 8, gw = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    unsigned acc = 0;
    for (uint64_t s0 = gw * G; s0 < nseg; s0 += nw * G) {
        const uint64_t s = s0 + grp < nseg ? s0 + grp : s0;
        const uint4* p = x + s * seg_vecs + sl;
        for (uint64_t j = 0; j < seg_vecs; j += LPS * DEPTH) {
            uint4 v[DEPTH];
#pragma unroll
            for (int d = 0; d < DEPTH; ++d) v[d] = ld(p + j + d * LPS);
#pragma unroll
            for (int d = 0; d < DEPTH; ++d) acc ^= v[d].x ^ v[d].y ^ v[d].z ^ v[d].w;
        }
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

template <typename F>
float timeit(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) f();
    cudaEventRecord(a);
    for (int i = 0; i < 20; ++i) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / 20;
}

int main() {
    const uint64_t n = 1ull << 28, nv = n / 2;
    uint4* x; unsigned* sink;
    cudaMalloc(&x, n * 8); cudaMalloc(&sink, 4);
    cudaMemset(x, 1, n * 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto rep = [&](const char* what, float ms) { printf("%-40s %8.1f us  %7.1f GB/s\n", what, ms * 1e3, n * 8 / ms / 1e6); };
    rep("grid-stride depth 4", timeit([&] { k_grid<4><<<2 * sms, 256>>>(x, nv, sink); }));
    rep("grid-stride depth 8", timeit([&] { k_grid<8><<<2 * sms, 256>>>(x, nv, sink); }));
    for (uint64_t L : {1024ull, 4096ull, 65536ull}) {
        uint64_t nseg = n / L, sv = L / 2;
        char buf[64];
        unsigned g = (unsigned)((nseg + 7) / 8 < (uint64_t)2 * sms ? (nseg + 7) / 8 : 2 * sms);
        snprintf(buf, 64, "warp/segment L=%llu depth 4", (unsigned long long)L);
        rep(buf, timeit([&] { k_seg<4><<<g, 256>>>(x, nseg, sv, sink); }));
        snprintf(buf, 64, "warp/segment L=%llu depth 8", (unsigned long long)L);
        rep(buf, timeit([&] { k_seg<8><<<g, 256>>>(x, nseg, sv, sink); }));
        unsigned g2 = (unsigned)((nseg + 15) / 16 < (uint64_t)2 * sms ? (nseg + 15) / 16 : 2 * sms);
        snprintf(buf, 64, "half-warp/segment L=%llu depth 8", (unsigned long long)L);
        rep(buf, timeit([&] { k_seg_part<8, 16><<<g2, 256>>>(x, nseg, sv, sink); }));
        snprintf(buf, 64, "half-warp/segment L=%llu depth 16", (unsigned long long)L);
        rep(buf, timeit([&] { k_seg_part<16, 16><<<g2, 256>>>(x, nseg, sv, sink); }));
        unsigned g4 = (unsigned)((nseg + 31) / 32 < (uint64_t)2 * sms ? (nseg + 31) / 32 : 2 * sms);
        snprintf(buf, 64, "quarter-warp/segment L=%llu depth 16", (unsigned long long)L);
        rep(buf, timeit([&] { k_seg_part<16, 8><<<g4, 256>>>(x, nseg, sv, sink); }));
        if (L >= 4096) {
            snprintf(buf, 64, "warp/segment L=%llu depth 16", (unsigned long long)L);
            rep(buf, timeit([&] { k_seg<16><<<g, 256>>>(x, nseg, sv, sink); }));
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
