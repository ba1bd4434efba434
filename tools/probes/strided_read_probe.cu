// Read-bandwidth probe of K10's access pattern (development tool, standalone): a [4096, 65536]
// binary64 matrix reduced over dim 0; one lane per column i, a warp covers 32 consecutive columns,
// 16 warps per block on neighbouring column groups; rows streamed with DEPTH rows in flight per lane.
// Variants: 8-B loads (one column per lane, as K10) and 16-B loads (two columns per lane).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o strided_read_probe strided_read_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <typename V>
__device__ __forceinline__ V ld(const V* p) { return __ldg(p); }

template <int DEPTH, typename V>
__global__ void __launch_bounds__(512, 1) k_cols(const V* x, uint64_t rows, uint64_t inner_v, unsigned* sink) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t groups = inner_v / 32;
    unsigned acc = 0;
    for (uint64_t g = (uint64_t)blockIdx.x * 16 + warp; g < groups; g += (uint64_t)gridDim.x * 16) {
        const V* q = x + g * 32 + lane;
        for (uint64_t r = 0; r < rows; r += DEPTH) {
            V v[DEPTH];
#pragma unroll
            for (int d = 0; d < DEPTH; ++d) v[d] = ld(q + (r + d) * inner_v);
#pragma unroll
            for (int d = 0; d < DEPTH; ++d) {
                const unsigned* w = reinterpret_cast<const unsigned*>(&v[d]);
#pragma unroll
                for (int k = 0; k < (int)(sizeof(V) / 4); ++k) acc ^= w[k];
            }
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
    const uint64_t rows = 4096, cols = 65536, n = rows * cols;
    double* x; unsigned* sink;
    cudaMalloc(&x, n * 8); cudaMalloc(&sink, 4);
    cudaMemset(x, 1, n * 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto rep = [&](const char* what, float ms) { printf("%-44s %8.1f us  %7.1f GB/s\n", what, ms * 1e3, n * 8 / ms / 1e6); };
    rep("8-B lanes (K10), depth 8, 1 block/SM", timeit([&] { k_cols<8, unsigned long long><<<sms, 512>>>((const unsigned long long*)x, rows, cols, sink); }));
    rep("8-B lanes (K10), depth 16", timeit([&] { k_cols<16, unsigned long long><<<sms, 512>>>((const unsigned long long*)x, rows, cols, sink); }));
    rep("8-B lanes (K10), depth 32", timeit([&] { k_cols<32, unsigned long long><<<sms, 512>>>((const unsigned long long*)x, rows, cols, sink); }));
    rep("16-B lanes (2 columns), depth 8", timeit([&] { k_cols<8, uint4><<<sms, 512>>>((const uint4*)x, rows, cols / 2, sink); }));
    rep("16-B lanes (2 columns), depth 16", timeit([&] { k_cols<16, uint4><<<sms, 512>>>((const uint4*)x, rows, cols / 2, sink); }));
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
