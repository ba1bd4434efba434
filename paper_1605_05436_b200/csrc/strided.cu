// K10: exact reductions along a strided dimension ("exact reduction along a
// tensor dim"): x viewed as [outer][len][inner] (inner > 1), out[o][i] = RN-even of the exact
// sum over r of x[o][r][i], with no transposing copy.
//
// Every lane owns one fibre (o, i) and its private 42-digit column in shared memory - the same
// lane column as K2 (the whole superaccumulator in internal memory,
// components added in any order; chunks of PAPER.md:744-750). A warp covers 32 consecutive i,
// so each row step is one coalesced 32-element load. Because the 32 columns of a warp belong
// to 32 different sums, each lane canonicalizes and rounds its own column sequentially
// (PAPER.md:777-795 steps 6-7 done by one thread) instead of the warp-cooperative finalize.
// When outer * ceil(inner/32) warps cannot fill the GPU, the rows are split into P parts whose
// regularized columns go to a caller-provided work buffer and are merged digit-wise by a second
// kernel (the Lemma-1 merge of PAPER.md:559-576, here a plain digit sum of P <= 1024 regularized
// columns followed by one regularization), which then rounds.
#include <cuda_runtime.h>

#include "lane_round.cuh"
#include "xsum_device.cuh"
#include "xsum_kernels.h"

namespace xs {

constexpr int STR_WARPS = 16;             // one 512-thread block per SM (168 KiB of columns)
#ifndef XS_STR_UNR
#define XS_STR_UNR 8
#endif
constexpr int STR_UNR = XS_STR_UNR;       // rows loaded together per lane (one group)
#ifndef XS_STR_NB
#define XS_STR_NB 4
#endif
constexpr int STR_NB = XS_STR_NB;         // rotating group buffers
constexpr size_t STR_SMEM = (size_t)STR_WARPS * D * 32 * sizeof(int64_t);

// Round the lane's regularized column and store fibre f's outputs (specials per R10).
__device__ __forceinline__ void lane_store(int64_t* col, uint32_t flags, const StrOut& o, uint64_t f) {
    const LaneTop t = lane_canonical_top(col);
    uint32_t rf = 0;
    uint64_t b64 = o.out64 ? lane_round(t, 53, 0, 2047, true, rf) : 0;
    uint32_t b32 = o.out32 ? (uint32_t)lane_round(t, 24, 925, 255, false, rf) : 0;
    const uint32_t fl = (flags & (XSUM_F_NAN | XSUM_F_PINF | XSUM_F_NINF)) | rf;
    if ((fl & XSUM_F_NAN) || ((fl & XSUM_F_PINF) && (fl & XSUM_F_NINF))) {
        b64 = 0x7FF8000000000000ull; b32 = 0x7FC00000u;
    } else if (fl & XSUM_F_PINF) {
        b64 = 0x7FF0000000000000ull; b32 = 0x7F800000u;
    } else if (fl & XSUM_F_NINF) {
        b64 = 0xFFF0000000000000ull; b32 = 0xFF800000u;
    }
    if (o.out64) o.out64[f] = __longlong_as_double((long long)b64);
    if (o.out32) o.out32[f] = __uint_as_float(b32);
    if (o.flags) o.flags[f] = fl;
}

template <int DT>
__global__ void __launch_bounds__(STR_WARPS * 32, 1)
k_sum_strided(const typename StrLd<DT>::T* __restrict__ x, uint64_t outer, uint64_t len, uint64_t inner,
              uint32_t parts, StrOut o, int64_t* __restrict__ work, uint32_t* __restrict__ wflags, uint32_t one,
              uint32_t mone) {
    using L = StrLd<DT>;
    extern __shared__ __align__(16) int64_t win[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t* col = win + warp * (D * 32) + lane;
    const uint64_t gpr = (inner + 31) / 32;                    // warps per outer row
    const uint64_t items = outer * gpr * parts;
    const uint64_t plen = (len + parts - 1) / parts;           // rows per part
    const uint64_t F = outer * inner;
    for (uint64_t it = (uint64_t)blockIdx.x * STR_WARPS + warp; it < items; it += (uint64_t)gridDim.x * STR_WARPS) {
        const uint64_t p = it % parts, grp = it / parts;
        const uint64_t ob = grp / gpr, i = (grp % gpr) * 32 + lane;
        const bool act = i < inner;
        const uint64_t r0 = p * plen < len ? p * plen : len;
        const uint64_t r1 = r0 + plen < len ? r0 + plen : len;
#pragma unroll
        for (int j = 0; j < D; ++j) col[j * 32] = 0;
        uint32_t flags = 0;
        if (act) {
            const typename L::T* q = x + (ob * len + r0) * inner + i;
            const typename L::T* qw = q;                       // window start (rows rw..r)
            uint64_t r = r0, rw = r0;
            int since = 0;
            uint32_t nspec = 0;
            // NaN/Inf patterns are added unchecked as if finite (their chunks stay inside the
            // window) and tracked by a running max of the exponent index; a window that saw one
            // is re-read and those chunks cancelled exactly (K2's rare path, per lane).
            auto close_window = [&]() {
                if (spec_hit(nspec)) {                         // rare: waits for the loads in flight
                    regularize_column(col);
                    const typename L::T* qq = qw;
                    for (uint64_t rr = rw; rr < r; ++rr, qq += inner) {
                        L::fix(col, L::raw(qq), flags, one);
                    }
                }
                regularize_column_inl(col);
                nspec = 0;
                since = 0;
                rw = r;
                qw = q;
            };
            // groups of STR_UNR rows through STR_NB rotating register buffers: STR_NB-1 groups
            // in flight while one is added (K2's scheme; one batch at a time measured 3 TB/s)
            const uint64_t ngroups = (r1 - r0) / STR_UNR;
            typename L::R buf[STR_NB][STR_UNR];
            const typename L::T* lq = q;
            uint64_t lg = 0;
#pragma unroll
            for (int b = 0; b < STR_NB - 1; ++b) {
                if (lg < ngroups) {
#pragma unroll
                    for (int u = 0; u < STR_UNR; ++u) buf[b][u] = L::raw(lq + u * inner);
                    lq += STR_UNR * inner;
                    ++lg;
                }
            }
            for (uint64_t g = 0; g < ngroups;) {
#pragma unroll
                for (int b = 0; b < STR_NB; ++b) {
                    if (g >= ngroups) break;
                    if (lg < ngroups) {
#pragma unroll
                        for (int u = 0; u < STR_UNR; ++u) buf[(b + STR_NB - 1) % STR_NB][u] = L::raw(lq + u * inner);
                        lq += STR_UNR * inner;
                        ++lg;
                    }
#pragma unroll
                    for (int u = 0; u < STR_UNR; ++u) {
                        Chunks c = L::dec(buf[b][u], one, mone);
                        nspec = spec_fold(nspec, c);
                        column_add(col, c, one);
                    }
                    q += STR_UNR * inner;
                    r += STR_UNR;
                    ++g;
                    since += STR_UNR;
                    if (since > FLUSH_ELEMS - STR_UNR) close_window();   // per-lane headroom (K2's window)
                }
            }
            for (; r < r1;) {
                const typename L::R v = L::raw(q);
                q += inner;
                ++r;
                Chunks c = L::dec(v, one, mone);
                nspec = spec_fold(nspec, c);
                column_add(col, c, one);
            }
            close_window();
            const uint64_t f = ob * inner + i;
            if (parts == 1) {
                lane_store(col, flags, o, f);
            } else {                                           // partial column -> work[p][j][f]
#pragma unroll 6
                for (int j = 0; j < D; ++j) work[(p * D + j) * F + f] = col[j * 32];
                wflags[p * F + f] = flags;
            }
        }
    }
}

// Merge of the P partial columns of 32 fibres per block: warp w sums parts w, w+16, ... in
// registers (42 coalesced loads per part), the 16 warp sums meet in shared memory, warp 0 adds
// them (|sum| <= P (2^51 + 1) < 2^62 for P <= 1024), regularizes and rounds each lane's fibre.
__global__ void __launch_bounds__(STR_WARPS * 32, 1)
k_strided_merge(const int64_t* __restrict__ work, const uint32_t* __restrict__ wflags, uint64_t F, uint32_t parts,
                StrOut o) {
    extern __shared__ __align__(16) int64_t win[];
    __shared__ uint32_t wfl[STR_WARPS][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t f = (uint64_t)blockIdx.x * 32 + lane;
    const bool act = f < F;
    int64_t acc[D];
#pragma unroll
    for (int j = 0; j < D; ++j) acc[j] = 0;
    uint32_t flags = 0;
    if (act) {
        for (uint32_t p = warp; p < parts; p += STR_WARPS) {
            flags |= wflags[p * F + f];
#pragma unroll
            for (int j = 0; j < D; ++j) acc[j] += work[(p * D + j) * F + f];
        }
    }
    int64_t* col = win + warp * (D * 32) + lane;
#pragma unroll
    for (int j = 0; j < D; ++j) col[j * 32] = acc[j];
    wfl[warp][lane] = flags;
    __syncthreads();
    if (warp != 0 || !act) return;
    for (int w = 1; w < STR_WARPS; ++w) {
        flags |= wfl[w][lane];
#pragma unroll 6
        for (int j = 0; j < D; ++j) col[j * 32] += win[w * (D * 32) + j * 32 + lane];
    }
    regularize_column(col);
    lane_store(col, flags, o, f);
}

// Row split: P parts per fibre group. Cost model in units of one full-GPU pass over the input:
// the wave quantization of outer*ceil(inner/32)*P warp items over the resident warp slots, plus
// the partial columns' extra traffic (written and read once, 336 B per fibre and part) relative
// to the input bytes.
uint32_t strided_parts(uint64_t outer, uint64_t len, uint64_t inner, int num_sms) {
    const uint64_t warps = outer * ((inner + 31) / 32);
    const uint64_t slots = (uint64_t)num_sms * STR_WARPS;
    if (warps == 0 || len < 512) return 1;
    uint64_t pmax = len / 256;
    if (pmax > 1024) pmax = 1024;
    const double in_bytes = (double)outer * (double)len * (double)inner * 2.0;   // >= 2 B per element
    const double per_part = 2.0 * (double)(D * 8 + 4) * (double)(outer * inner) / in_bytes;
    uint64_t best = 1;
    double best_cost = 1e300;
    for (uint64_t p = 1; p <= pmax; p = p < 64 ? p + 1 : p + p / 8) {
        const double items = (double)(warps * p);
        const double waves = (double)((warps * p + slots - 1) / slots);
        const double cost = waves * (double)slots / items + (p > 1 ? per_part * (double)p : 0.0);
        if (cost < best_cost - 1e-9) { best_cost = cost; best = p; }
    }
    return (uint32_t)best;
}

size_t strided_work_bytes(uint64_t outer, uint64_t len, uint64_t inner, int num_sms) {
    const uint32_t p = strided_parts(outer, len, inner, num_sms);
    return p > 1 ? (size_t)p * outer * inner * (D * sizeof(int64_t) + sizeof(uint32_t)) : 0;
}

template <int DT>
static cudaError_t launch_strided(const void* x, uint64_t outer, uint64_t len, uint64_t inner, uint32_t parts,
                                  const StrOut& o, int64_t* work, uint32_t* wflags, int num_sms, cudaStream_t s) {
    static unsigned long long done = 0;
    if (cudaError_t e = ensure_smem(k_sum_strided<DT>, STR_SMEM, done)) return e;
    const uint64_t items = outer * ((inner + 31) / 32) * parts;
    const uint64_t want = (items + STR_WARPS - 1) / STR_WARPS;
    const unsigned g = (unsigned)(want < (uint64_t)num_sms ? want : num_sms);
    k_sum_strided<DT><<<g, STR_WARPS * 32, STR_SMEM, s>>>(static_cast<const typename StrLd<DT>::T*>(x), outer, len,
                                                          inner, parts, o, work, wflags, 1u, 0xFFFFFFFFu);
    note_launch();
    return cudaGetLastError();
}

cudaError_t sum_strided(const void* x, int dtype, uint64_t outer, uint64_t len, uint64_t inner, const StrOut& o,
                        void* work, size_t work_bytes, int num_sms, cudaStream_t s) {
    if (outer == 0 || inner == 0) return cudaSuccess;
    uint32_t parts = strided_parts(outer, len, inner, num_sms);
    if (parts > 1 && (!work || work_bytes < strided_work_bytes(outer, len, inner, num_sms))) parts = 1;
    const uint64_t F = outer * inner;
    int64_t* wk = parts > 1 ? static_cast<int64_t*>(work) : nullptr;
    uint32_t* wf = parts > 1 ? reinterpret_cast<uint32_t*>(wk + (size_t)parts * D * F) : nullptr;
    cudaError_t e;
    switch (dtype) {
        case XSUM_DT_F64: e = launch_strided<XSUM_DT_F64>(x, outer, len, inner, parts, o, wk, wf, num_sms, s); break;
        case XSUM_DT_F32: e = launch_strided<XSUM_DT_F32>(x, outer, len, inner, parts, o, wk, wf, num_sms, s); break;
        case XSUM_DT_F16: e = launch_strided<XSUM_DT_F16>(x, outer, len, inner, parts, o, wk, wf, num_sms, s); break;
        default: e = launch_strided<XSUM_DT_BF16>(x, outer, len, inner, parts, o, wk, wf, num_sms, s); break;
    }
    if (e != cudaSuccess || parts == 1) return e;
    static unsigned long long done_m = 0;
    if ((e = ensure_smem(k_strided_merge, STR_SMEM, done_m))) return e;
    const unsigned gm = (unsigned)((F + 31) / 32);
    k_strided_merge<<<gm, STR_WARPS * 32, STR_SMEM, s>>>(wk, wf, F, parts, o);
    note_launch();
    return cudaGetLastError();
}

}  // namespace xs
