// Internal launcher interface between the C-ABI (api.cu) and the kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "xsum.h"

#define XS_MAXB 1024   // max blocks of one accumulate launch (1024 x regularized partials < 2^62)

namespace xs {

// Fused multi-GPU step (SURVEY.md §8(e) fused option): the exchange buffers of the `world`
// ranks, addressable by every rank (NVLink P2P / symmetric memory). Buffer layout:
// [2][world][XSUM_STATE_BYTES] state slots (parity of the call's epoch) then a u64 arrival
// counter that every rank's call increments once (monotone: epoch e is complete at e*world).
struct PeerParams {
    uint8_t* const* bufs;      // device array of the world buffer pointers (null: no exchange)
    uint32_t rank, world;
    uint64_t epoch;            // 1, 2, 3, ... per call on the same buffers
};
constexpr size_t peer_counter_off(uint32_t world) { return 2ull * world * XSUM_STATE_BYTES; }
constexpr size_t peer_buffer_bytes(uint32_t world) { return peer_counter_off(world) + 64; }

struct AccParams {
    xsum_state_image* state;   // handle state (device)
    int64_t* gacc;             // [D] grid accumulator: every block red.adds its partial (scratch, 0 between launches)
    uint32_t* gflags;          // grid flags (red.or; scratch, 0 between launches)
    uint32_t* counter;         // arrival counter (scratch, 0 between launches)
    int64_t* stamps;           // XS_TIMING builds: [6][XS_MAXB] %globaltimer stamps (scratch), else null
    int overwrite;             // 1: state := sum (fused reset), 0: state += sum
    xsum_result* res;          // non-null: fused finalize
    uint64_t* canon;           // optional canonical image for the fused finalize
    uint32_t one;              // = 1  } opaque to the compiler: keeps selected integer ops as IMADs
    uint32_t mone;             // = -1 } on the FMA pipe instead of ALU-pipe IADD3s
    PeerParams peer;           // fused cross-GPU exchange after the grid merge (bufs null: none)
    const uint32_t* skip;      // non-null: the launch does nothing if *skip != 0 when it starts (read
                               // after the predecessor completed; K12's exact pass)
};

// XS_TIMING=1: diagnostic builds (tools/timing_probe.py) stamp %globaltimer per block; 0 in the product
#ifndef XS_TIMING
#define XS_TIMING 0
#endif
// scratch layout: [0,4) arrival counter, [4,8) grid flags; [256, 256 + 8 D) grid accumulator;
// timing builds only: [1024, 1024 + 8 * 6 * MAXB) stamps
constexpr size_t SCRATCH_COUNTER_OFF = 0;
constexpr size_t SCRATCH_GFLAGS_OFF = 4;
constexpr size_t SCRATCH_ACC_OFF = 256;
constexpr size_t SCRATCH_STAMP_OFF = 1024;
constexpr size_t SCRATCH_BYTES = SCRATCH_STAMP_OFF + (XS_TIMING ? sizeof(int64_t) * 6 * XS_MAXB : 0);

void note_launch();

// Programmatic dependent launch (sm_90+): an accumulate launch may place its blocks on SMs while
// the previous kernel in the stream is still finishing (its last block merging and rounding,
// slower SMs streaming their last tiles); each block zeroes its lane columns and then waits for
// the predecessor's completion (griddepcontrol.wait) BEFORE its first input load. A predecessor
// may signal its dependents early (e.g. GEMM kernels before their epilogue stores) and its
// writes are only guaranteed visible after griddepcontrol.wait, so reading the input earlier
// would be unsafe for arbitrary producers; the overlap kept is the launch and the
// block prologue. XSUM_NO_PDL=1 in the environment launches normally (A/B measurements). Only
// launches of less than PDL_MAX_BYTES of input use it.
bool pdl_enabled();
constexpr uint64_t PDL_MAX_BYTES = 1ull << 30;

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(bool pdl, void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem,
                              cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (pdl && pdl_enabled()) ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

__device__ __forceinline__ void pdl_release_dependents() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void pdl_wait_predecessor() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// XS_TIMING builds: stamp k of block b at stamps[k * XS_MAXB + b] (scratch).
__device__ __forceinline__ void xs_stamp(int64_t* stamps, int k, unsigned b) {
#if XS_TIMING
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    stamps[(size_t)k * XS_MAXB + b] = (int64_t)t;
#else
    (void)stamps; (void)k; (void)b;
#endif
}

// Opt `kernel` into `bytes` of dynamic shared memory once per device: the attribute belongs to
// the function in the current device's context, so a process driving several GPUs sets it on
// each. `done` is the caller's per-kernel bitmask of devices (device index < 64).
template <typename K>
inline cudaError_t ensure_smem(K kernel, size_t bytes, unsigned long long& done) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = 1ull << (dev & 63);
    if (__atomic_load_n(&done, __ATOMIC_ACQUIRE) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) __atomic_fetch_or(&done, bit, __ATOMIC_RELEASE);
    return e;
}

cudaError_t accumulate(const double* x, uint64_t n, const AccParams& p, int num_sms, cudaStream_t s);
cudaError_t accumulate_f32(const float* x, uint64_t n, const AccParams& p, int num_sms, cudaStream_t s);
cudaError_t accumulate_h16(const uint16_t* x, uint64_t n, int bf16, const AccParams& p, int num_sms, cudaStream_t s);
cudaError_t init_state(xsum_state_image* st, cudaStream_t s);
cudaError_t merge_states(xsum_state_image* st, const void* states, uint32_t count, int overwrite, xsum_result* res,
                         uint64_t* canon, cudaStream_t s);
cudaError_t merge_sparse(xsum_state_image* st, const void* images, const uint64_t* offsets, uint32_t count,
                         cudaStream_t s);
cudaError_t to_sparse(const xsum_state_image* st, void* out, uint32_t* nbytes, cudaStream_t s);
cudaError_t peer_selftest(const xsum_state_image* states, uint8_t* const* bufs, uint32_t world, uint64_t epoch,
                          xsum_result* res, xsum_state_image* out, cudaStream_t s);
cudaError_t finalize(const xsum_state_image* st, xsum_result* res, uint64_t* canon, cudaStream_t s);
// K12 (condsens.cu): the condition-number-sensitive iteration of PAPER.md:895-918
size_t condsens_work_bytes(uint64_t n);
cudaError_t condsens_sum(const double* x, uint64_t n, int rule, void* work, size_t work_bytes, xsum_result* res,
                         xsum_condsens_info* info, uint64_t* canon, int num_sms, cudaStream_t s);
// Per-segment outputs (any may be null): binary64 / binary32 roundings, canonical images, flags.
struct SegOut {
    double* out;
    float* out32;
    uint64_t* canon;
    uint32_t* flags;
    __device__ __forceinline__ void write(uint64_t s, const xsum_result& r) const {
        if (out) out[s] = r.value;
        if (out32) out32[s] = __uint_as_float(r.value_f32);
        if (flags) flags[s] = r.flags;
    }
};

// ticket: optional zeroed 8-byte device counter; with CSR offsets the warps draw segments from
// it (dynamic balancing of ragged lengths), else the static order s, s + nw, ...
cudaError_t sum_segments(const double* x, uint64_t nseg, uint64_t seg_len, const uint64_t* offsets, const SegOut& o,
                         int num_sms, cudaStream_t s, unsigned long long* ticket = nullptr);
// equal binary64 segments, half a warp per segment (K6h, segments_half.cu)
bool segments_half_ok(const double* x, uint64_t seg_len);
cudaError_t sum_segments_half(const double* x, uint64_t nseg, uint64_t seg_len, const SegOut& o, int num_sms,
                              cudaStream_t s);
// short equal segments, one lane per segment (K11, segments_lanes.cu); sum_segments and
// sum_segments_small route equal segments of length <= SEG_LANES_MAX here
#ifndef XS_SEG_LANES_MAX
#define XS_SEG_LANES_MAX 256
#endif
constexpr uint64_t SEG_LANES_MAX = XS_SEG_LANES_MAX;
cudaError_t sum_segments_lanes(const void* x, int dtype, uint64_t nseg, uint64_t len, const SegOut& o, int num_sms,
                               cudaStream_t s);
// CSR segments, mostly short: short ones one lane each, the rest by the warp (K11c)
cudaError_t sum_segments_lanes_csr(const void* x, int dtype, uint64_t nseg, const uint64_t* offsets, const SegOut& o,
                                   unsigned long long* ticket, int num_sms, cudaStream_t s);
// strided reductions (K10, strided.cu): x as [outer][len][inner], out[o*inner + i]
struct StrOut {
    double* out64;
    float* out32;
    uint32_t* flags;
};
uint32_t strided_parts(uint64_t outer, uint64_t len, uint64_t inner, int num_sms);
size_t strided_work_bytes(uint64_t outer, uint64_t len, uint64_t inner, int num_sms);
cudaError_t sum_strided(const void* x, int dtype, uint64_t outer, uint64_t len, uint64_t inner, const StrOut& o,
                        void* work, size_t work_bytes, int num_sms, cudaStream_t s);
// binary32 / binary16 / bfloat16 elements (dtype XSUM_DT_F32 / F16 / BF16), equal or CSR segments
cudaError_t sum_segments_small(const void* x, int dtype, uint64_t nseg, uint64_t seg_len, const uint64_t* offsets,
                               const SegOut& o, int num_sms, cudaStream_t s, unsigned long long* ticket = nullptr);

}  // namespace xs
