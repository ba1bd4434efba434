// Seeded synthetic inputs, device implementation (bench/test infrastructure).
//
// Holds none of the method's arithmetic: it writes binary64 bit patterns from the
// counter-based splitmix64 definition in synth/gen.py. It lets
// bench.py create the 2-64 GiB workloads in HBM in milliseconds. Tests check it
// bit for bit against synth/gen.py and synth/gen.c.
#include <cuda_runtime.h>
#include <stdint.h>

#define SYNTH_G 0x9E3779B97F4A7C15ull

__device__ __forceinline__ uint64_t s_mix64(uint64_t z) {
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27; z *= 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t s_draw(uint64_t key, uint64_t i, int lo, int hi) {
    uint64_t u = s_mix64(key + SYNTH_G * (2 * i + 1));
    uint64_t v = s_mix64(key + SYNTH_G * (2 * i + 2));
    uint64_t span = (uint64_t)(hi - lo + 1);
    uint64_t e = ((v >> 32) * span) >> 32;
    uint64_t biased = (uint64_t)((int64_t)e + lo + 1023);
    return (u & 0x8000000000000000ull) | (biased << 52) | (u & ((1ull << 52) - 1));
}

static uint64_t h_mix64(uint64_t z) {
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27; z *= 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static uint64_t h_key(uint64_t seed, uint64_t st) { return h_mix64(seed + SYNTH_G * (st + 1)); }

__global__ void k_uniform(uint64_t* __restrict__ out, uint64_t start, uint64_t count, uint64_t key,
                          int lo, int hi) {
    uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += stride)
        out[t] = s_draw(key, start + t, lo, hi);
}

__global__ void k_cancel(uint64_t* __restrict__ out, uint64_t start, uint64_t count, uint64_t ka,
                         uint64_t kt, uint64_t npairs, int plo, int phi, int tlo, int thi) {
    uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t n2 = 2 * npairs;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += stride) {
        uint64_t p = start + t;
        out[t] = p < n2 ? (s_draw(ka, p >> 1, plo, phi) ^ ((p & 1) << 63)) : s_draw(kt, p - n2, tlo, thi);
    }
}

// Keys for the c3 permutation, with the top bit flipped so that a signed int64 sort
// orders them as unsigned U(seed, st, idx).
__global__ void k_keys_signed(int64_t* __restrict__ out, uint64_t start, uint64_t count, uint64_t key) {
    uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += stride)
        out[t] = (int64_t)(s_mix64(key + SYNTH_G * (start + t + 1)) ^ 0x8000000000000000ull);
}

// Test helper (tests/test_gpu_api_r02.py): a producer that releases its programmatic dependents at
// entry (griddepcontrol.launch_dependents), waits ~spin cycles, then fills x[0..n) with v - like a
// GEMM that triggers its dependents before its epilogue stores. A PDL-launched consumer that read
// its input before griddepcontrol.wait would see the old contents.
__global__ void k_fill_after_trigger(double* x, uint64_t n, double v, long long spin) {
    asm volatile("griddepcontrol.launch_dependents;");
    const long long t0 = clock64();
    while (clock64() - t0 < spin) {
    }
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += stride) x[t] = v;
}

static unsigned grid_for(uint64_t count) {
    uint64_t b = (count + 255) / 256;
    return (unsigned)(b < 148ull * 64 ? (b ? b : 1) : 148ull * 64);
}

extern "C" {

int synth_gpu_uniform(void* out, uint64_t start, uint64_t count, uint64_t seed, uint64_t st, int lo,
                      int hi, void* stream) {
    if (!count) return 0;
    k_uniform<<<grid_for(count), 256, 0, (cudaStream_t)stream>>>((uint64_t*)out, start, count,
                                                                   h_key(seed, st), lo, hi);
    return (int)cudaGetLastError();
}

int synth_gpu_cancel_unpermuted(void* out, uint64_t start, uint64_t count, uint64_t seed,
                                uint64_t npairs, int plo, int phi, int tlo, int thi, void* stream) {
    if (!count) return 0;
    k_cancel<<<grid_for(count), 256, 0, (cudaStream_t)stream>>>(
        (uint64_t*)out, start, count, h_key(seed, 0), h_key(seed, 1), npairs, plo, phi, tlo, thi);
    return (int)cudaGetLastError();
}

int synth_gpu_keys_signed(void* out, uint64_t start, uint64_t count, uint64_t seed, uint64_t st,
                          void* stream) {
    if (!count) return 0;
    k_keys_signed<<<grid_for(count), 256, 0, (cudaStream_t)stream>>>((int64_t*)out, start, count,
                                                                       h_key(seed, st));
    return (int)cudaGetLastError();
}

int synth_gpu_fill_after_trigger(void* x, uint64_t n, double v, long long spin, void* stream) {
    if (!n) return 0;
    // a few small blocks: the producer must leave the other SMs free, or the consumer's blocks
    // could not become resident before it exits and the race would be hidden
    k_fill_after_trigger<<<4, 256, 0, (cudaStream_t)stream>>>((double*)x, n, v, spin);
    return (int)cudaGetLastError();
}

}  // extern "C"
