// K7: exact sums of 16-bit inputs, IEEE binary16 and bfloat16.
//
// The paper's format has a t-bit fraction and an l-bit exponent; binary16
// is t = 10, l = 5 and bfloat16 t = 7, l = 8 (IEEE bias, reading R1). Every such value is
// M 2^k in units of its least subnormal, M = m + [e!=0] 2^t < 2^(t+1), k = max(e,1) - 1.
// With so few significand bits the superaccumulator's components can be much narrower than
// the binary64 path's 52-bit digits (components are integers whose
// exponents are multiples of a fixed width): each lane keeps unsigned 32-bit "bins", one per
// (sign, exponent group) with groups of 2^SB consecutive exponents, and adds M 2^(k mod 2^SB)
// into the bin of its group - one 32-bit add per summand, no carries, no sign handling. Every
// FLUSH adds (before a bin can wrap) the bins are emptied into a narrow per-lane column of the
// 52-bit digits the format reaches (h16_common.cuh); at the end the columns are combined into
// digits and merged up the same grid tree as binary64 sums (grid_tail.cuh).
// NaN/Inf patterns fall into a
// bin group of their own (exponent field all ones) that is never summed: a lane that sees it
// non-empty at a window close rescans its window to classify NaN / +Inf / -Inf (reading R10).
#include <cuda_runtime.h>

#include "grid_tail.cuh"
#include "h16_common.cuh"
#include "xsum_device.cuh"
#include "xsum_kernels.h"

namespace xs {

constexpr int H16_WARPS = 16;
constexpr int H16_U = 4;          // 16-B vectors per thread per tile (8 summands each)
#ifndef XS_H16_NB
#define XS_H16_NB 4
#endif
constexpr int H16_NB = XS_H16_NB; // rotating register buffers (NB-1 tiles in flight)

template <class F>
__device__ __noinline__ void h16_rescan(const uint4* body, uint64_t t0, uint64_t t1, uint64_t G, uint64_t TV, int tid,
                                        uint32_t& flags) {
    // rare path: classify the NaN/Inf patterns of this lane's window (they were binned into
    // the special group, which is never summed)
    for (uint64_t tt = t0; tt <= t1; tt += G) {
        for (int u = 0; u < H16_U; ++u) {
            uint4 v = ld_stream(body + tt * TV + (uint64_t)u * (H16_WARPS * 32) + tid);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
            for (int i = 0; i < 4; ++i) flags |= h16_special_flags<F>(w[i] & 0xFFFFu) | h16_special_flags<F>(w[i] >> 16);
        }
    }
}

// Checked single summand (head / tail / leftovers): specials are flagged, not binned.
template <class F>
__device__ __forceinline__ void h16_add_checked(uint32_t* bins, uint32_t b16, uint32_t& flags) {
    const uint32_t f = h16_special_flags<F>(b16);
    if (f) { flags |= f; return; }
    h16_add<F>(bins, b16 & 0x7FFFu, b16 >> 15);
}

template <class F>
__global__ void __launch_bounds__(H16_WARPS * 32, 1)
k_accumulate_h16(const uint16_t* x, uint64_t n, AccParams p) {
    using C = H16Col<F>;
    constexpr int T = H16_WARPS * 32;
    constexpr int PV = 8;                                   // summands per 16-B vector
    constexpr int FLUSH_TILES = F::FLUSH / (PV * H16_U);    // tiles per bin window
    constexpr int GROUPS_PER_WINDOW = FLUSH_TILES / H16_NB;
    static_assert(GROUPS_PER_WINDOW >= 1, "window shorter than one buffer group");
    // per lane: NBIN u32 bins and a COLS-digit int64 column (thread-minor, conflict-free)
    extern __shared__ __align__(16) int64_t smem64[];
    int64_t* const cols_all = smem64;                                         // [WARPS][COLS][32]
    uint32_t* const bins_all = reinterpret_cast<uint32_t*>(smem64 + H16_WARPS * C::COLS * 32);
    __shared__ int64_t wsum[H16_WARPS][32];
    __shared__ int64_t digits[64];                          // grid-tail scratch
    __shared__ int64_t su[64];
    __shared__ uint32_t blk_flags;
    __shared__ int is_last;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    pdl_release_dependents();    // the next launch may take SMs as this grid's blocks finish
    uint32_t* bins = bins_all + warp * (F::NBIN * 32) + lane;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(bins);
    const uint32_t sbase2 = sbase * 0x00010001u;
    const uint32_t one = p.one, mone = p.mone;
    int64_t* col = cols_all + warp * (C::COLS * 32) + lane;
#pragma unroll
    for (int b = 0; b < F::NBIN; ++b) bins[b * 32] = 0;
#pragma unroll
    for (int j = 0; j < C::COLS; ++j) col[j * 32] = 0;
    if (tid == 0) blk_flags = 0;
    uint32_t flags = 0;
    pdl_wait_predecessor();      // inputs are read only after the preceding launch completed

    // peel up to 7 head elements to reach 16-B alignment; <= 7 tail elements remain
    uint64_t head = ((16 - ((uintptr_t)x & 15)) & 15) / 2;
    if (head > n) head = n;
    const uint64_t nbody = n - head;
    const uint64_t nvec = nbody / PV;
    const uint4* body = reinterpret_cast<const uint4*>(x + head);
    const uint64_t TV = (uint64_t)T * H16_U;
    const uint64_t ntiles = nvec / TV;
    const uint64_t G = gridDim.x;

    uint64_t wstart = blockIdx.x, tlast = 0;
    bool any_tile = false;
    int flushes = 0;
    auto load_tile = [&](uint4 (&buf)[H16_U], uint64_t tt) {
        if (tt < ntiles) {
#pragma unroll
            for (int u = 0; u < H16_U; ++u) buf[u] = ld_stream(body + tt * TV + (uint64_t)u * T + tid);
        }
    };
    uint4 buf[H16_NB][H16_U];
    uint64_t t = blockIdx.x;
#pragma unroll
    for (int b = 0; b < H16_NB; ++b) load_tile(buf[b], t + (uint64_t)b * G);
    bool more = t < ntiles;
    int groups = 0;
    while (more) {
#pragma unroll
        for (int b = 0; b < H16_NB; ++b) {
            if (more) {
#pragma unroll
                for (int u = 0; u < H16_U; ++u) {
                    h16_add_word<F>(sbase, sbase2, buf[b][u].x, one, mone);
                    h16_add_word<F>(sbase, sbase2, buf[b][u].y, one, mone);
                    h16_add_word<F>(sbase, sbase2, buf[b][u].z, one, mone);
                    h16_add_word<F>(sbase, sbase2, buf[b][u].w, one, mone);
                }
                any_tile = true;
                tlast = t;
                load_tile(buf[b], t + (uint64_t)H16_NB * G);
                t += G;
                more = t < ntiles;
            }
        }
        if (++groups == GROUPS_PER_WINDOW) {
            if (h16_flush_col<F>(bins, col)) h16_rescan<F>(body, wstart, tlast, G, TV, tid, flags);
            if (++flushes == C::REG_FLUSHES) { h16_col_regularize<F>(col); flushes = 0; }
            groups = 0;
            wstart = t;
            any_tile = false;
        }
    }
    if (h16_flush_col<F>(bins, col) && any_tile) h16_rescan<F>(body, wstart, tlast, G, TV, tid, flags);

    // leftover vectors (< one tile), the unaligned head and the tail: checked adds by the block
    // that would own the next tile (<= 4 vectors + 1 element per thread: no bin can wrap)
    if (blockIdx.x == ntiles % G) {
        const uint64_t v0 = ntiles * TV;
        for (int u = 0; u < H16_U; ++u) {
            uint64_t v = v0 + (uint64_t)u * T + tid;
            if (v < nvec) {
                uint4 q = ld_stream(body + v);
                const uint32_t w[4] = {q.x, q.y, q.z, q.w};
                for (int i = 0; i < 4; ++i) {
                    h16_add_checked<F>(bins, w[i] & 0xFFFFu, flags);
                    h16_add_checked<F>(bins, w[i] >> 16, flags);
                }
            }
        }
        const uint64_t tail = nbody - nvec * PV;
        if ((uint64_t)tid < head) h16_add_checked<F>(bins, ld_coherent(x + tid), flags);
        if (tid >= 8 && (uint64_t)(tid - 8) < tail) h16_add_checked<F>(bins, ld_coherent(x + head + nvec * PV + (tid - 8)), flags);
    }
    h16_flush_col<F>(bins, col);
    __syncwarp();

    // warp: the 32 narrow columns become the warp's digits (lane j: digit j); block: warp 0 sums
    // the warps (|.| <= 16 (2^51 + 2^16)) and regularizes; grid: grid_tail.cuh
    {
        wsum[warp][lane] = h16_col_combine<F>(cols_all + warp * (C::COLS * 32), lane);
        const uint32_t f = __reduce_or_sync(FULL, flags);
        if (lane == 0 && f) atomicOr(&blk_flags, f);
    }
    __syncthreads();
    int64_t a0 = 0, a1 = 0;
    if (warp == 0) {
#pragma unroll
        for (int w = 0; w < H16_WARPS; ++w) a0 += wsum[w][lane];
        regularize_warp(a0, a1, lane);
    }
    grid_tail<H16_WARPS>(a0, a1, blk_flags, n, p, digits, su, &blk_flags, &is_last, warp, lane);
}

template <class F>
static cudaError_t launch_h16(const uint16_t* x, uint64_t n, const AccParams& p, int num_sms, cudaStream_t s) {
    constexpr size_t SMEM = (size_t)H16_WARPS * 32 * (H16Col<F>::COLS * 8 + F::NBIN * 4);
    static unsigned long long smem_set = 0;
    if (cudaError_t e = ensure_smem(k_accumulate_h16<F>, SMEM, smem_set)) return e;
    uint64_t head = ((16 - ((uintptr_t)x & 15)) & 15) / 2;
    if (head > n) head = n;
    const uint64_t ntiles = ((n - head) / 8) / ((uint64_t)H16_WARPS * 32 * H16_U);
    uint64_t g = ntiles < (uint64_t)num_sms ? ntiles : (uint64_t)num_sms;
    if (g < 1) g = 1;
    if (g > XS_MAXB) g = XS_MAXB;
    cudaError_t e = launch_pdl(n * 2 < PDL_MAX_BYTES, k_accumulate_h16<F>, (unsigned)g, H16_WARPS * 32, SMEM, s, x, n, p);
    note_launch();
    return e;
}

cudaError_t accumulate_h16(const uint16_t* x, uint64_t n, int bf16, const AccParams& p, int num_sms, cudaStream_t s) {
    return bf16 ? launch_h16<FmtBF16>(x, n, p, num_sms, s) : launch_h16<FmtF16>(x, n, p, num_sms, s);
}

}  // namespace xs
