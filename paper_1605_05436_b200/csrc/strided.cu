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

#include "f32_bins.cuh"
#include "h16_common.cuh"
#include "lane_round.cuh"
#include "xsum_device.cuh"
#include "xsum_kernels.h"

namespace xs {

constexpr int STR_WARPS = 16;             // one 512-thread block per SM (168 KiB of columns)
#ifndef XS_STRH
#define XS_STRH 1                         // 16-bit strided reductions through K10h (tools/variants.py: 0)
#endif
#ifndef XS_STR_UNR
#define XS_STR_UNR 8
#endif
constexpr int STR_UNR = XS_STR_UNR;       // rows loaded together per lane (one group)
#ifndef XS_STR_NB
#define XS_STR_NB 4
#endif
constexpr int STR_NB = XS_STR_NB;         // rotating group buffers
constexpr size_t STR_SMEM = (size_t)STR_WARPS * D * 32 * sizeof(int64_t);
#ifndef XS_STR_SK
#define XS_STR_SK 1                       // binary64 strided reductions through K10s when it balances better
#endif

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

// Rows [r0, r1) of fibre (ob, i) into the lane's (zeroed) column, leaving it regularized; NaN / Inf
// flags into `flags`.
template <int DT>
__device__ __forceinline__ void strided_rows(const typename StrLd<DT>::T* __restrict__ x, uint64_t ob, uint64_t i,
                                             uint64_t len, uint64_t inner, uint64_t r0, uint64_t r1, int64_t* col,
                                             uint32_t& flags, uint32_t one, uint32_t mone) {
    using L = StrLd<DT>;
    {
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
    }
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
        const uint64_t p = it / (items / parts), grp = it % (items / parts);   // neighbouring warps: neighbouring fibres
        const uint64_t ob = grp / gpr, i = (grp % gpr) * 32 + lane;
        const bool act = i < inner;
        const uint64_t r0 = p * plen < len ? p * plen : len;
        const uint64_t r1 = r0 + plen < len ? r0 + plen : len;
#pragma unroll
        for (int j = 0; j < D; ++j) col[j * 32] = 0;
        uint32_t flags = 0;
        if (act) {
            strided_rows<DT>(x, ob, i, len, inner, r0, r1, col, flags, one, mone);
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

// K10s bookkeeping (K10s and its narrow-format kernels): a piece's rows join its group's count after
// its accumulator adds (fence first); true on every lane for the piece that completes the group.
__device__ __forceinline__ bool sk_piece_done(uint32_t* cnt, uint64_t rows, uint64_t len, int lane) {
    __threadfence();
    __syncwarp();
    uint32_t last = 0;
    if (lane == 0) last = atomicAdd(cnt, (uint32_t)rows) + (uint32_t)rows == (uint32_t)len;
    last = __shfl_sync(FULL, last, 0);
    if (last) __threadfence();
    return last != 0;
}
// The item loop: SK = stream-K (every resident warp an equal share of groups x len row units, in
// order; whole groups mode 0, pieces mode 2), else (part, group) items (mode 0 for one part, 1 for
// a part of several).
template <bool SK, int WARPS, class Fn>
__device__ __forceinline__ void sk_or_parts(uint64_t groups, uint64_t len, uint32_t parts, uint64_t plen,
                                            uint64_t items, int lane, int warp, Fn&& range) {
    (void)lane;
    if constexpr (SK) {
        const uint64_t U = groups * len;
        const uint64_t nw = (uint64_t)gridDim.x * WARPS, w = (uint64_t)blockIdx.x * WARPS + warp;
        uint64_t u0 = (uint64_t)(((unsigned __int128)U * w) / nw);
        const uint64_t u1 = (uint64_t)(((unsigned __int128)U * (w + 1)) / nw);
        while (u0 < u1) {
            const uint64_t grp = u0 / len, r0 = u0 - grp * len;
            const uint64_t r1 = r0 + (u1 - u0) < len ? r0 + (u1 - u0) : len;
            range(grp, r0, r1, 0, (r0 == 0 && r1 == len) ? 0 : 2);
            u0 += r1 - r0;
        }
    } else {
    for (uint64_t it = (uint64_t)blockIdx.x * WARPS + warp; it < items; it += (uint64_t)gridDim.x * WARPS) {
        const uint64_t p = it / (items / parts), grp = it % (items / parts);   // neighbouring warps: neighbouring fibres
        const uint64_t r0 = p * plen < len ? p * plen : len;
        const uint64_t r1 = r0 + plen < len ? r0 + plen : len;
        range(grp, r0, r1, p, parts == 1 ? 0 : 1);
    }
    }
}

// K10s: the same lane-per-fibre reduction, stream-K ordered (round 2). When outer * ceil(inner/32)
// warp items do not fill the resident warps evenly (c2dim0: 2048 items on 148 x 16 = 2368 slots,
// 20 SMs idle for the whole launch), every resident warp takes an equal share of the rows of all
// fibre groups in order, [u0, u1) of outer * ceil(inner/32) * len row units: a warp finishes at most
// one group it started elsewhere and starts at most one it does not finish. A group summed by one
// warp is rounded at once; the pieces of a split group add their regularized columns into a
// per-fibre accumulator (acc[j][f], L2-resident red.add; |digit| stays below 2^55 for the <= len
// pieces a group can have) and count their rows; the piece whose rows complete the group reads the
// accumulator back, regularizes and rounds. acc, the flag words and the counters are zero on entry
// (the launch clears them first).
template <int DT>
__global__ void __launch_bounds__(STR_WARPS * 32, 1)
k_sum_strided_sk(const typename StrLd<DT>::T* __restrict__ x, uint64_t outer, uint64_t len, uint64_t inner,
                 StrOut o, int64_t* __restrict__ acc, uint32_t* __restrict__ aflags, uint32_t* __restrict__ cnt,
                 uint32_t one, uint32_t mone) {
    extern __shared__ __align__(16) int64_t win[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t* col = win + warp * (D * 32) + lane;
    const uint64_t gpr = (inner + 31) / 32;
    const uint64_t F = outer * inner;
    auto range = [&](uint64_t grp, uint64_t r0, uint64_t r1, uint64_t, int mode) {
        const uint64_t ob = grp / gpr, i = (grp % gpr) * 32 + lane;
        const bool act = i < inner;
        const uint64_t f = ob * inner + i;
#pragma unroll
        for (int j = 0; j < D; ++j) col[j * 32] = 0;
        uint32_t flags = 0;
        if (act) strided_rows<DT>(x, ob, i, len, inner, r0, r1, col, flags, one, mone);
        if (mode == 2) {                                       // a piece: add into acc[j][f]
            if (act) {
#pragma unroll 6
                for (int j = 0; j < D; ++j)
                    atomicAdd(reinterpret_cast<unsigned long long*>(acc + (uint64_t)j * F + f),
                              (unsigned long long)col[j * 32]);
                if (flags) atomicOr(aflags + f, flags);
            }
            if (!sk_piece_done(cnt + grp, r1 - r0, len, lane)) return;
            if (act) {                                         // this piece completes the group
#pragma unroll 6
                for (int j = 0; j < D; ++j)
                    col[j * 32] = __ldcg(reinterpret_cast<const long long*>(acc + (uint64_t)j * F + f));
                flags = __ldcg(aflags + f);
                regularize_column(col);
            }
        }
        if (act) lane_store(col, flags, o, f);
    };
    sk_or_parts<true, STR_WARPS>(outer * gpr, len, 1, len, outer * gpr, lane, warp, range);
}

// Stream-K pays off when the warp items leave resident warp slots idle (a wave-quantization loss
// above 4%) and len fits the 32-bit row counters; its work: acc [D][F] int64 + flags [F] + counters.
static bool strided_sk_wanted(uint64_t outer, uint64_t len, uint64_t inner, int num_sms, uint64_t fpw = 32) {
    const uint64_t items = outer * ((inner + fpw - 1) / fpw), slots = (uint64_t)num_sms * STR_WARPS;
    if (items == 0 || len < 64 || len >= (1ull << 31)) return false;
    const uint64_t waves = (items + slots - 1) / slots;
    return (double)(waves * slots - items) > 0.04 * (double)(waves * slots);
}
static size_t strided_sk_bytes(uint64_t outer, uint64_t inner) {
    const uint64_t F = outer * inner, groups = outer * ((inner + 31) / 32);
    return (size_t)F * (D * sizeof(int64_t) + sizeof(uint32_t)) + (size_t)groups * sizeof(uint32_t);
}

// ---------------------------------------------------------------------------------------------
// K10h: binary16 / bfloat16 strided reductions, TWO fibres per lane: a lane loads one 32-bit word
// per row (fibres i, i+1; 128 B per warp per row) and decodes both halves at once into per-fibre
// 32-bit exponent-group bins (K7's packed decode, h16_common.cuh; one red.shared per element
// instead of K10's two 64-bit read-modify-writes of a 42-digit column), emptied into narrow
// per-fibre digit columns every window; each lane rounds its two fibres with the carry chain of
// K11 (lane_top_chain) on the narrow column. NaN/Inf patterns land in a group that is never
// summed; a lane that saw one re-reads its fibres to classify them (R10). Partial columns of a
// row split are widened to K10's 42-digit layout and merged by k_strided_merge.
// ---------------------------------------------------------------------------------------------
constexpr int STRH_WARPS = 16;
#ifndef XS_STRH_UNR
#define XS_STRH_UNR 16        // rows per group for the narrow kernels (8: bfloat16 545, binary32 715 G/s; 16: 569 / 838)
#endif
#ifndef XS_STRH_NB
#define XS_STRH_NB 4
#endif
constexpr int STRH_UNR = XS_STRH_UNR, STRH_NB = XS_STRH_NB;
// K10h rows per group: bfloat16 8 (its kernel is large enough for instruction-cache stalls at 16:
// 1477 vs 1430 G/s on [4096, 65536] over dim 0), binary16 16 (1755 vs 1586 at 8)
template <class F>
constexpr int strh_unr() { return F::t == 7 ? 8 : STRH_UNR; }
template <class F>
constexpr size_t strh_smem() {
    return (size_t)STRH_WARPS * 32 * 2 * (H16Col<F>::COLS * 8 + F::NBIN * 4);
}

template <class F>
__device__ __noinline__ uint32_t strh_classify(const uint16_t* q, uint64_t rows, uint64_t inner) {
    uint32_t f = 0;
    for (uint64_t r = 0; r < rows; ++r) f |= h16_special_flags<F>(__ldg(q + r * inner));
    return f;
}

template <class F>
__device__ __forceinline__ void strh_store(int64_t* col, uint32_t flags, const StrOut& o, uint64_t f) {
    using C = H16Col<F>;
    LaneTop t = lane_top_chain<32>(col, 0, C::COLS - 1);       // zeroes the column
    if (t.m >= 0) t.m += C::COL0;
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

template <class F>
__global__ void __launch_bounds__(STRH_WARPS * 32, 1)
k_sum_strided_h16(const uint16_t* __restrict__ x, uint64_t outer, uint64_t len, uint64_t inner, uint32_t parts,
                  StrOut o, int64_t* __restrict__ work, uint32_t* __restrict__ wflags, uint32_t one, uint32_t mone) {
    using C = H16Col<F>;
    constexpr int HU = strh_unr<F>();                          // rows per group
    extern __shared__ __align__(16) int64_t win[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t* const colw = win + warp * (2 * C::COLS * 32);
    int64_t* col[2] = {colw + lane, colw + C::COLS * 32 + lane};
    uint32_t* const binw = reinterpret_cast<uint32_t*>(win + STRH_WARPS * 2 * C::COLS * 32) + warp * (2 * F::NBIN * 32);
    uint32_t* bins[2] = {binw + lane, binw + F::NBIN * 32 + lane};
    const uint32_t sb0 = (uint32_t)__cvta_generic_to_shared(bins[0]);
    const uint32_t sb1 = (uint32_t)__cvta_generic_to_shared(bins[1]);
    const uint32_t sb2 = sb0 + (sb1 << 16);                     // low half -> fibre i, high half -> i + 1
    constexpr uint32_t WIN = (uint32_t)(F::FLUSH / HU) * HU;   // rows per bin window
    const uint64_t gpr = (inner + 63) / 64;
    const uint64_t items = outer * gpr * parts;
    const uint64_t plen = (len + parts - 1) / parts;
    const uint64_t Fn = outer * inner;
    const uint64_t wstride = inner / 2;                           // 32-bit words per row
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int j = 0; j < C::COLS; ++j) col[h][j * 32] = 0;
#pragma unroll
        for (int j = 0; j < F::NBIN; ++j) bins[h][j * 32] = 0;
    }
    for (uint64_t it = (uint64_t)blockIdx.x * STRH_WARPS + warp; it < items; it += (uint64_t)gridDim.x * STRH_WARPS) {
        const uint64_t p = it / (items / parts), grp = it % (items / parts);   // neighbouring warps: neighbouring fibres
        const uint64_t ob = grp / gpr, i = (grp % gpr) * 64 + 2 * (uint64_t)lane;
        const bool act = i < inner;                                // inner is even: both fibres or none
        const uint64_t r0 = p * plen < len ? p * plen : len;
        const uint64_t r1 = r0 + plen < len ? r0 + plen : len;
        bool special = false;
        uint32_t flushes = 0;
        if (act) {
            const uint32_t* q = reinterpret_cast<const uint32_t*>(x + (ob * len + r0) * inner + i);
            const uint64_t ngroups = (r1 - r0) / HU;
            uint32_t buf[STRH_NB][HU];
            const uint32_t* lq = q;
            uint64_t lg = 0;
#pragma unroll
            for (int b = 0; b < STRH_NB - 1; ++b) {
                if (lg < ngroups) {
#pragma unroll
                    for (int u = 0; u < HU; ++u) buf[b][u] = __ldcs(lq + u * wstride);
                    lq += HU * wstride;
                    ++lg;
                }
            }
            uint32_t since = 0;
            for (uint64_t g = 0; g < ngroups;) {
#pragma unroll
                for (int b = 0; b < STRH_NB; ++b) {
                    if (g >= ngroups) break;
                    if (lg < ngroups) {
#pragma unroll
                        for (int u = 0; u < HU; ++u)
                            buf[(b + STRH_NB - 1) % STRH_NB][u] = __ldcs(lq + u * wstride);
                        lq += HU * wstride;
                        ++lg;
                    }
#pragma unroll
                    for (int u = 0; u < HU; ++u) h16_add_word<F>(sb1, sb2, buf[b][u], one, mone);
                    ++g;
                    since += HU;
                    if (since == WIN) {                          // bin window full: empty into the columns
                        special |= h16_flush_col<F>(bins[0], col[0]);
                        special |= h16_flush_col<F>(bins[1], col[1]);
                        since = 0;
                        if (++flushes == C::REG_FLUSHES) {
                            h16_col_regularize<F>(col[0]);
                            h16_col_regularize<F>(col[1]);
                            flushes = 0;
                        }
                    }
                }
            }
            for (uint64_t r = r0 + ngroups * HU; r < r1; ++r) {   // < HU rows left: in the window
                h16_add_word<F>(sb1, sb2, __ldcs(q + (r - r0) * wstride), one, mone);
            }
            special |= h16_flush_col<F>(bins[0], col[0]);
            special |= h16_flush_col<F>(bins[1], col[1]);
        }
        uint32_t fl[2] = {0, 0};
        if (special) {                                             // rare: classify this lane's fibres
            const uint16_t* q16 = x + (ob * len + r0) * inner + i;
            fl[0] = strh_classify<F>(q16, r1 - r0, inner);
            fl[1] = strh_classify<F>(q16 + 1, r1 - r0, inner);
        }
        if (act) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint64_t f = ob * inner + i + h;
                if (parts == 1) {
                    strh_store<F>(col[h], fl[h], o, f);
                } else {                                           // partial -> work[p][j][f], 42 digits
                    h16_col_regularize<F>(col[h]);
                    for (int j = 0; j < D; ++j) {
                        const int r = j - C::COL0;
                        int64_t v = 0;
                        if (r >= 0 && r < C::COLS) {
                            v = col[h][r * 32];
                            col[h][r * 32] = 0;
                        }
                        work[(p * D + j) * Fn + f] = v;
                    }
                    wflags[p * Fn + f] = fl[h];
                }
            }
        }
    }
}

// K10s for K10h: the kernel above as stream-K pieces (sk_or_parts<true>: modes 0 and 2 only). One
// templated body for both made ptxas spill 230-370 B in the row-parts instantiation (the lambda's
// captures), so the stream-K form is a separate kernel.
template <class F>
__global__ void __launch_bounds__(STRH_WARPS * 32, 1)
k_sum_strided_h16_sk(const uint16_t* __restrict__ x, uint64_t outer, uint64_t len, uint64_t inner, uint32_t parts,
                  StrOut o, int64_t* __restrict__ work, uint32_t* __restrict__ wflags, uint32_t* __restrict__ cnt,
                  uint32_t one, uint32_t mone) {
    using C = H16Col<F>;
    constexpr int HU = strh_unr<F>();                          // rows per group
    extern __shared__ __align__(16) int64_t win[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t* const colw = win + warp * (2 * C::COLS * 32);
    int64_t* col[2] = {colw + lane, colw + C::COLS * 32 + lane};
    uint32_t* const binw = reinterpret_cast<uint32_t*>(win + STRH_WARPS * 2 * C::COLS * 32) + warp * (2 * F::NBIN * 32);
    uint32_t* bins[2] = {binw + lane, binw + F::NBIN * 32 + lane};
    const uint32_t sb0 = (uint32_t)__cvta_generic_to_shared(bins[0]);
    const uint32_t sb1 = (uint32_t)__cvta_generic_to_shared(bins[1]);
    const uint32_t sb2 = sb0 + (sb1 << 16);                     // low half -> fibre i, high half -> i + 1
    constexpr uint32_t WIN = (uint32_t)(F::FLUSH / HU) * HU;   // rows per bin window
    const uint64_t gpr = (inner + 63) / 64;
    const uint64_t items = outer * gpr * parts;
    const uint64_t plen = (len + parts - 1) / parts;
    const uint64_t Fn = outer * inner;
    const uint64_t wstride = inner / 2;                           // 32-bit words per row
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int j = 0; j < C::COLS; ++j) col[h][j * 32] = 0;
#pragma unroll
        for (int j = 0; j < F::NBIN; ++j) bins[h][j * 32] = 0;
    }
    // mode 0: whole fibres (round and store); 1: a row part -> work[p]; 2: a stream-K piece (K10s).
    // (the pointer arrays by copy: a by-reference capture put them in local memory, 230 B of spills)
    auto range = [&, col, bins](uint64_t grp, uint64_t r0, uint64_t r1, uint64_t p, int mode) {
        const uint64_t ob = grp / gpr, i = (grp % gpr) * 64 + 2 * (uint64_t)lane;
        const bool act = i < inner;                                // inner is even: both fibres or none
        bool special = false;
        uint32_t flushes = 0;
        if (act) {
            const uint32_t* q = reinterpret_cast<const uint32_t*>(x + (ob * len + r0) * inner + i);
            const uint64_t ngroups = (r1 - r0) / HU;
            uint32_t buf[STRH_NB][HU];
            const uint32_t* lq = q;
            uint64_t lg = 0;
#pragma unroll
            for (int b = 0; b < STRH_NB - 1; ++b) {
                if (lg < ngroups) {
#pragma unroll
                    for (int u = 0; u < HU; ++u) buf[b][u] = __ldcs(lq + u * wstride);
                    lq += HU * wstride;
                    ++lg;
                }
            }
            uint32_t since = 0;
            for (uint64_t g = 0; g < ngroups;) {
#pragma unroll
                for (int b = 0; b < STRH_NB; ++b) {
                    if (g >= ngroups) break;
                    if (lg < ngroups) {
#pragma unroll
                        for (int u = 0; u < HU; ++u)
                            buf[(b + STRH_NB - 1) % STRH_NB][u] = __ldcs(lq + u * wstride);
                        lq += HU * wstride;
                        ++lg;
                    }
#pragma unroll
                    for (int u = 0; u < HU; ++u) h16_add_word<F>(sb1, sb2, buf[b][u], one, mone);
                    ++g;
                    since += HU;
                    if (since == WIN) {                          // bin window full: empty into the columns
                        special |= h16_flush_col<F>(bins[0], col[0]);
                        special |= h16_flush_col<F>(bins[1], col[1]);
                        since = 0;
                        if (++flushes == C::REG_FLUSHES) {
                            h16_col_regularize<F>(col[0]);
                            h16_col_regularize<F>(col[1]);
                            flushes = 0;
                        }
                    }
                }
            }
            for (uint64_t r = r0 + ngroups * HU; r < r1; ++r) {   // < HU rows left: in the window
                h16_add_word<F>(sb1, sb2, __ldcs(q + (r - r0) * wstride), one, mone);
            }
            special |= h16_flush_col<F>(bins[0], col[0]);
            special |= h16_flush_col<F>(bins[1], col[1]);
        }
        uint32_t fl[2] = {0, 0};
        if (special) {                                             // rare: classify this lane's fibres
            const uint16_t* q16 = x + (ob * len + r0) * inner + i;
            fl[0] = strh_classify<F>(q16, r1 - r0, inner);
            fl[1] = strh_classify<F>(q16 + 1, r1 - r0, inner);
        }
        if (mode == 2) {                                           // stream-K piece: add into acc[r][f]
            if (act) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint64_t f = ob * inner + i + h;
                    h16_col_regularize<F>(col[h]);
                    for (int r = 0; r < C::COLS; ++r) {
                        atomicAdd(reinterpret_cast<unsigned long long*>(work + (uint64_t)r * Fn + f),
                                  (unsigned long long)col[h][r * 32]);
                        col[h][r * 32] = 0;
                    }
                    if (fl[h]) atomicOr(wflags + f, fl[h]);
                }
            }
            if (!sk_piece_done(cnt + grp, r1 - r0, len, lane)) return;
            if (act) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint64_t f = ob * inner + i + h;
                    for (int r = 0; r < C::COLS; ++r)
                        col[h][r * 32] = __ldcg(reinterpret_cast<const long long*>(work + (uint64_t)r * Fn + f));
                    fl[h] = __ldcg(wflags + f);
                }
            }
            mode = 0;
        }
        if (act) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint64_t f = ob * inner + i + h;
                if (mode == 0) {
                    strh_store<F>(col[h], fl[h], o, f);
                } else {                                  // partial -> work[p][j][f], 42 digits
                    h16_col_regularize<F>(col[h]);
                    for (int j = 0; j < D; ++j) {
                        const int r = j - C::COL0;
                        int64_t v = 0;
                        if (r >= 0 && r < C::COLS) {
                            v = col[h][r * 32];
                            col[h][r * 32] = 0;
                        }
                        work[(p * D + j) * Fn + f] = v;
                    }
                    wflags[p * Fn + f] = fl[h];
                }
            }
        }
    };
    sk_or_parts<true, STRH_WARPS>(outer * gpr, len, parts, plen, items, lane, warp, range);
}

// ---------------------------------------------------------------------------------------------
// K10f: binary32 strided reductions with K9's 64-bit exponent-group bins (f32_bins.cuh): one 64-bit
// read-modify-write per element instead of K10's two (the element's two 52-bit digit chunks),
// emptied into a narrow column every window; each lane rounds its fibre with the carry chain.
// NaN/Inf patterns are summed as finite and, if a lane saw one, cancelled by a rescan of its fibre
// (the sign-flipped pattern lands in the other sign's bin of the same group).
// ---------------------------------------------------------------------------------------------
template <class F>
constexpr size_t strf_smem() {
    return (size_t)STR_WARPS * 32 * (F::COLS + F::NBIN) * 8;
}

template <class F>
__device__ __noinline__ void strf_rescan(uint64_t* bins, int64_t* col, const uint32_t* q, uint64_t rows,
                                         uint64_t inner, uint32_t& flags, uint32_t one) {
    uint32_t dummy = 0, adds = 0, flushes = 0;
    scol_regularize<F>(col);
    for (uint64_t r = 0; r < rows; ++r) {
        const uint32_t b = __ldg(q + r * inner);
        const uint32_t f = sspecial_flags<F>(b);
        if (f) {
            flags |= f;
            sbin_add<F>(bins, b ^ (1u << (F::t + F::l)), dummy, one);
            if (++adds == SSEG_FLUSH) {
                sbin_flush<F>(bins, col);
                adds = 0;
                if (++flushes == SSEG_REG_FLUSHES) { scol_regularize<F>(col); flushes = 0; }
            }
        }
    }
    sbin_flush<F>(bins, col);
}

template <class F>
__global__ void __launch_bounds__(STR_WARPS * 32, 1)
k_sum_strided_f32(const uint32_t* __restrict__ x, uint64_t outer, uint64_t len, uint64_t inner, uint32_t parts,
                  StrOut o, int64_t* __restrict__ work, uint32_t* __restrict__ wflags, uint32_t one) {
    extern __shared__ __align__(16) int64_t win[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t* col = win + warp * (F::COLS * 32) + lane;
    uint64_t* bins = reinterpret_cast<uint64_t*>(win + STR_WARPS * F::COLS * 32) + warp * (F::NBIN * 32) + lane;
    constexpr uint32_t WIN = (uint32_t)(SSEG_FLUSH / STRH_UNR) * STRH_UNR;    // rows per bin window
    const uint64_t gpr = (inner + 31) / 32;
    const uint64_t items = outer * gpr * parts;
    const uint64_t plen = (len + parts - 1) / parts;
    const uint64_t Fn = outer * inner;
#pragma unroll
    for (int j = 0; j < F::COLS; ++j) col[j * 32] = 0;
#pragma unroll
    for (int j = 0; j < F::NBIN; ++j) bins[j * 32] = 0;
    for (uint64_t it = (uint64_t)blockIdx.x * STR_WARPS + warp; it < items; it += (uint64_t)gridDim.x * STR_WARPS) {
        const uint64_t p = it / (items / parts), grp = it % (items / parts);   // neighbouring warps: neighbouring fibres
        const uint64_t ob = grp / gpr, i = (grp % gpr) * 32 + lane;
        const bool act = i < inner;
        const uint64_t r0 = p * plen < len ? p * plen : len;
        const uint64_t r1 = r0 + plen < len ? r0 + plen : len;
        uint32_t flags = 0;
        if (act) {
            const uint32_t* q = x + (ob * len + r0) * inner + i;
            const uint64_t ngroups = (r1 - r0) / STRH_UNR;
            uint32_t buf[STRH_NB][STRH_UNR];
            const uint32_t* lq = q;
            uint64_t lg = 0;
            uint32_t spec = 0, since = 0, flushes = 0;
#pragma unroll
            for (int b = 0; b < STRH_NB - 1; ++b) {
                if (lg < ngroups) {
#pragma unroll
                    for (int u = 0; u < STRH_UNR; ++u) buf[b][u] = __ldcs(lq + u * inner);
                    lq += STRH_UNR * inner;
                    ++lg;
                }
            }
            for (uint64_t g = 0; g < ngroups;) {
#pragma unroll
                for (int b = 0; b < STRH_NB; ++b) {
                    if (g >= ngroups) break;
                    if (lg < ngroups) {
#pragma unroll
                        for (int u = 0; u < STRH_UNR; ++u) buf[(b + STRH_NB - 1) % STRH_NB][u] = __ldcs(lq + u * inner);
                        lq += STRH_UNR * inner;
                        ++lg;
                    }
#pragma unroll
                    for (int u = 0; u < STRH_UNR; ++u) sbin_add<F>(bins, buf[b][u], spec, one);
                    ++g;
                    since += STRH_UNR;
                    if (since == WIN) {
                        sbin_flush<F>(bins, col);
                        since = 0;
                        if (++flushes == SSEG_REG_FLUSHES) { scol_regularize<F>(col); flushes = 0; }
                    }
                }
            }
            for (uint64_t r = r0 + ngroups * STRH_UNR; r < r1; ++r) sbin_add<F>(bins, __ldcs(q + (r - r0) * inner), spec, one);
            sbin_flush<F>(bins, col);
            if (spec == F::EM) strf_rescan<F>(bins, col, q, r1 - r0, inner, flags, one);   // rare
            const uint64_t f = ob * inner + i;
            if (parts == 1) {
                LaneTop t = lane_top_chain<32>(col, 0, F::COLS - 1);    // zeroes the column
                if (t.m >= 0) t.m += F::COL0;
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
            } else {                                             // partial -> work[p][j][f], 42 digits
                scol_regularize<F>(col);
                for (int j = 0; j < D; ++j) {
                    const int r = j - F::COL0;
                    int64_t v = 0;
                    if (r >= 0 && r < F::COLS) {
                        v = col[r * 32];
                        col[r * 32] = 0;
                    }
                    work[(p * D + j) * Fn + f] = v;
                }
                wflags[p * Fn + f] = flags;
            }
        }
    }
}

// K10s for K10f: the kernel above as stream-K pieces (sk_or_parts<true>: modes 0 and 2 only; a
// separate kernel for the same reason as k_sum_strided_h16_sk).
template <class F>
__global__ void __launch_bounds__(STR_WARPS * 32, 1)
k_sum_strided_f32_sk(const uint32_t* __restrict__ x, uint64_t outer, uint64_t len, uint64_t inner, uint32_t parts,
                  StrOut o, int64_t* __restrict__ work, uint32_t* __restrict__ wflags, uint32_t* __restrict__ cnt,
                  uint32_t one) {
    extern __shared__ __align__(16) int64_t win[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t* col = win + warp * (F::COLS * 32) + lane;
    uint64_t* bins = reinterpret_cast<uint64_t*>(win + STR_WARPS * F::COLS * 32) + warp * (F::NBIN * 32) + lane;
    constexpr uint32_t WIN = (uint32_t)(SSEG_FLUSH / STRH_UNR) * STRH_UNR;    // rows per bin window
    const uint64_t gpr = (inner + 31) / 32;
    const uint64_t items = outer * gpr * parts;
    const uint64_t plen = (len + parts - 1) / parts;
    const uint64_t Fn = outer * inner;
#pragma unroll
    for (int j = 0; j < F::COLS; ++j) col[j * 32] = 0;
#pragma unroll
    for (int j = 0; j < F::NBIN; ++j) bins[j * 32] = 0;
    // mode 0: the whole fibre (round and store); 1: a row part -> work[p]; 2: a stream-K piece (K10s)
    auto range = [&](uint64_t grp, uint64_t r0, uint64_t r1, uint64_t p, int mode) {
        const uint64_t ob = grp / gpr, i = (grp % gpr) * 32 + lane;
        const bool act = i < inner;
        uint32_t flags = 0;
        if (act) {
            const uint32_t* q = x + (ob * len + r0) * inner + i;
            const uint64_t ngroups = (r1 - r0) / STRH_UNR;
            uint32_t buf[STRH_NB][STRH_UNR];
            const uint32_t* lq = q;
            uint64_t lg = 0;
            uint32_t spec = 0, since = 0, flushes = 0;
#pragma unroll
            for (int b = 0; b < STRH_NB - 1; ++b) {
                if (lg < ngroups) {
#pragma unroll
                    for (int u = 0; u < STRH_UNR; ++u) buf[b][u] = __ldcs(lq + u * inner);
                    lq += STRH_UNR * inner;
                    ++lg;
                }
            }
            for (uint64_t g = 0; g < ngroups;) {
#pragma unroll
                for (int b = 0; b < STRH_NB; ++b) {
                    if (g >= ngroups) break;
                    if (lg < ngroups) {
#pragma unroll
                        for (int u = 0; u < STRH_UNR; ++u) buf[(b + STRH_NB - 1) % STRH_NB][u] = __ldcs(lq + u * inner);
                        lq += STRH_UNR * inner;
                        ++lg;
                    }
#pragma unroll
                    for (int u = 0; u < STRH_UNR; ++u) sbin_add<F>(bins, buf[b][u], spec, one);
                    ++g;
                    since += STRH_UNR;
                    if (since == WIN) {
                        sbin_flush<F>(bins, col);
                        since = 0;
                        if (++flushes == SSEG_REG_FLUSHES) { scol_regularize<F>(col); flushes = 0; }
                    }
                }
            }
            for (uint64_t r = r0 + ngroups * STRH_UNR; r < r1; ++r) sbin_add<F>(bins, __ldcs(q + (r - r0) * inner), spec, one);
            sbin_flush<F>(bins, col);
            if (spec == F::EM) strf_rescan<F>(bins, col, q, r1 - r0, inner, flags, one);   // rare
        }
        const uint64_t f = ob * inner + i;
        if (mode == 2) {                                         // stream-K piece: add into acc[r][f]
            if (act) {
                scol_regularize<F>(col);
                for (int r = 0; r < F::COLS; ++r) {
                    atomicAdd(reinterpret_cast<unsigned long long*>(work + (uint64_t)r * Fn + f),
                              (unsigned long long)col[r * 32]);
                    col[r * 32] = 0;
                }
                if (flags) atomicOr(wflags + f, flags);
            }
            if (!sk_piece_done(cnt + grp, r1 - r0, len, lane)) return;
            if (act) {
                for (int r = 0; r < F::COLS; ++r) col[r * 32] = __ldcg(reinterpret_cast<const long long*>(work + (uint64_t)r * Fn + f));
                flags = __ldcg(wflags + f);
            }
            mode = 0;
        }
        if (act) {
            if (mode == 0) {
                LaneTop t = lane_top_chain<32>(col, 0, F::COLS - 1);    // zeroes the column
                if (t.m >= 0) t.m += F::COL0;
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
            } else {                                    // partial -> work[p][j][f], 42 digits
                scol_regularize<F>(col);
                for (int j = 0; j < D; ++j) {
                    const int r = j - F::COL0;
                    int64_t v = 0;
                    if (r >= 0 && r < F::COLS) {
                        v = col[r * 32];
                        col[r * 32] = 0;
                    }
                    work[(p * D + j) * Fn + f] = v;
                }
                wflags[p * Fn + f] = flags;
            }
        }
    };
    sk_or_parts<true, STR_WARPS>(outer * gpr, len, parts, plen, items, lane, warp, range);
}

// sk: K10s (stream-K pieces meeting in work = acc [COLS][F], wflags [F], cnt [groups], cleared by the
// caller); else row parts (parts == 1: one item per fibre group).
template <class F>
static cudaError_t launch_strided_f32(const void* x, uint64_t outer, uint64_t len, uint64_t inner, uint32_t parts,
                                      const StrOut& o, int64_t* work, uint32_t* wflags, uint32_t* cnt, bool sk,
                                      int num_sms, cudaStream_t s) {
    static unsigned long long done = 0, done_sk = 0;
    if (cudaError_t e = ensure_smem(k_sum_strided_f32<F>, strf_smem<F>(), done)) return e;
    if (cudaError_t e = ensure_smem(k_sum_strided_f32_sk<F>, strf_smem<F>(), done_sk)) return e;
    const uint64_t items = outer * ((inner + 31) / 32) * parts;
    const uint64_t want = (items + STR_WARPS - 1) / STR_WARPS;
    const unsigned g = sk ? (unsigned)num_sms : (unsigned)(want < (uint64_t)num_sms ? want : num_sms);
    if (sk)
        k_sum_strided_f32_sk<F><<<g, STR_WARPS * 32, strf_smem<F>(), s>>>(static_cast<const uint32_t*>(x), outer, len,
                                                                          inner, 1, o, work, wflags, cnt, 1u);
    else
        k_sum_strided_f32<F><<<g, STR_WARPS * 32, strf_smem<F>(), s>>>(static_cast<const uint32_t*>(x), outer, len,
                                                                       inner, parts, o, work, wflags, 1u);
    note_launch();
    return cudaGetLastError();
}

template <class F>
static cudaError_t launch_strided_h16(const void* x, uint64_t outer, uint64_t len, uint64_t inner, uint32_t parts,
                                      const StrOut& o, int64_t* work, uint32_t* wflags, uint32_t* cnt, bool sk,
                                      int num_sms, cudaStream_t s) {
    static unsigned long long done = 0, done_sk = 0;
    if (cudaError_t e = ensure_smem(k_sum_strided_h16<F>, strh_smem<F>(), done)) return e;
    if (cudaError_t e = ensure_smem(k_sum_strided_h16_sk<F>, strh_smem<F>(), done_sk)) return e;
    const uint64_t items = outer * ((inner + 63) / 64) * parts;
    const uint64_t want = (items + STRH_WARPS - 1) / STRH_WARPS;
    const unsigned g = sk ? (unsigned)num_sms : (unsigned)(want < (uint64_t)num_sms ? want : num_sms);
    if (sk)
        k_sum_strided_h16_sk<F><<<g, STRH_WARPS * 32, strh_smem<F>(), s>>>(static_cast<const uint16_t*>(x), outer,
                                                                           len, inner, 1, o, work, wflags, cnt, 1u,
                                                                           0xFFFFFFFFu);
    else
        k_sum_strided_h16<F><<<g, STRH_WARPS * 32, strh_smem<F>(), s>>>(static_cast<const uint16_t*>(x), outer, len,
                                                                        inner, parts, o, work, wflags, 1u,
                                                                        0xFFFFFFFFu);
    note_launch();
    return cudaGetLastError();
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

// The same merge with one lane per fibre and no cross-warp step, for many fibres: each lane adds
// its fibre's P partial columns (coalesced across the warp) into its shared-memory column,
// regularizes and rounds. 4 warps and 42 KiB per block, so many blocks share an SM; the 16-warp
// kernel above (parts split across warps) stays for few fibres with many parts.
constexpr int STRM_WARPS = 4;
__global__ void __launch_bounds__(STRM_WARPS * 32)
k_strided_merge_lanes(const int64_t* __restrict__ work, const uint32_t* __restrict__ wflags, uint64_t F,
                      uint32_t parts, StrOut o) {
    __shared__ int64_t win[STRM_WARPS * D * 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t f = ((uint64_t)blockIdx.x * STRM_WARPS + warp) * 32 + lane;
    if (f >= F) return;
    int64_t* col = win + warp * (D * 32) + lane;
    int64_t acc[D];
#pragma unroll
    for (int j = 0; j < D; ++j) acc[j] = 0;
    uint32_t flags = 0;
    for (uint32_t p = 0; p < parts; ++p) {
        flags |= wflags[p * F + f];
#pragma unroll
        for (int j = 0; j < D; ++j) acc[j] += work[(p * D + j) * F + f];
    }
#pragma unroll
    for (int j = 0; j < D; ++j) col[j * 32] = acc[j];
    regularize_column(col);
    lane_store(col, flags, o, f);
}

// Row split: P parts per fibre group. Cost model in units of one full-GPU pass over the input:
// the wave quantization of outer*ceil(inner/32)*P warp items over the resident warp slots, plus
// the partial columns' extra traffic (written and read once, 336 B per fibre and part) relative
// to the input bytes.
static uint32_t parts_for(uint64_t outer, uint64_t len, uint64_t inner, int num_sms, uint64_t fpw) {
    const uint64_t warps = outer * ((inner + fpw - 1) / fpw);
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
uint32_t strided_parts(uint64_t outer, uint64_t len, uint64_t inner, int num_sms) {
    return parts_for(outer, len, inner, num_sms, 32);
}
// K10h (16-bit, two fibres per lane) covers 64 fibres per warp: fewer warp items, more parts
static uint32_t strided_parts_h16(uint64_t outer, uint64_t len, uint64_t inner, int num_sms) {
    return parts_for(outer, len, inner, num_sms, 64);
}

// The work buffer serves every element format (the size query has no dtype): the larger of the
// 32- and 64-fibre-per-warp splits.
size_t strided_work_bytes(uint64_t outer, uint64_t len, uint64_t inner, int num_sms) {
    uint32_t p = strided_parts(outer, len, inner, num_sms);
    const uint32_t ph = strided_parts_h16(outer, len, inner, num_sms);
    if (ph > p) p = ph;
    size_t b = p > 1 ? (size_t)p * outer * inner * (D * sizeof(int64_t) + sizeof(uint32_t)) : 0;
    if (XS_STR_SK && (strided_sk_wanted(outer, len, inner, num_sms) || strided_sk_wanted(outer, len, inner, num_sms, 64)) &&
        strided_sk_bytes(outer, inner) > b)
        b = strided_sk_bytes(outer, inner);                     // K10s
    return b;
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
    // 16-bit formats with an even inner size on a 4-B aligned base: two fibres per lane (K10h)
    const bool h16 = XS_STRH && (dtype == XSUM_DT_F16 || dtype == XSUM_DT_BF16) && inner % 2 == 0 &&
                     ((uintptr_t)x & 3) == 0;
    uint32_t parts = h16 ? strided_parts_h16(outer, len, inner, num_sms) : strided_parts(outer, len, inner, num_sms);
    if (parts > 1 && (!work || work_bytes < strided_work_bytes(outer, len, inner, num_sms))) parts = 1;
    const uint64_t F = outer * inner;
    // K10s for the narrow formats (K10h / K10f) whenever their items fill the resident warps unevenly
    const bool narrow = h16 || (dtype == XSUM_DT_F32 && XS_STRH);
    const bool skn = XS_STR_SK && narrow && work && strided_sk_wanted(outer, len, inner, num_sms, h16 ? 64 : 32) &&
                     work_bytes >= strided_sk_bytes(outer, inner);
    if (skn) parts = 1;
    int64_t* wk = parts > 1 ? static_cast<int64_t*>(work) : nullptr;
    uint32_t* wf = parts > 1 ? reinterpret_cast<uint32_t*>(wk + (size_t)parts * D * F) : nullptr;
    uint32_t* cnt = nullptr;
    cudaError_t e;
    if (skn) {
        const size_t nb = strided_sk_bytes(outer, inner);
        if ((e = cudaMemsetAsync(work, 0, nb, s))) return e;
        wk = static_cast<int64_t*>(work);
        wf = reinterpret_cast<uint32_t*>(wk + (size_t)D * F);
        cnt = wf + F;
    }
    if (h16) {
        e = dtype == XSUM_DT_F16
                ? launch_strided_h16<FmtF16>(x, outer, len, inner, parts, o, wk, wf, cnt, skn, num_sms, s)
                : launch_strided_h16<FmtBF16Q>(x, outer, len, inner, parts, o, wk, wf, cnt, skn, num_sms, s);
        if (skn) return e;
    } else if (skn) {
        return launch_strided_f32<SF32>(x, outer, len, inner, parts, o, wk, wf, cnt, true, num_sms, s);
    } else switch (dtype) {
        case XSUM_DT_F64:
            if (XS_STR_SK && parts == 1 && work && strided_sk_wanted(outer, len, inner, num_sms) &&
                work_bytes >= strided_sk_bytes(outer, inner)) {
                const size_t nb = strided_sk_bytes(outer, inner);
                if ((e = cudaMemsetAsync(work, 0, nb, s))) return e;
                static unsigned long long done_sk = 0;
                if ((e = ensure_smem(k_sum_strided_sk<XSUM_DT_F64>, STR_SMEM, done_sk))) return e;
                int64_t* acc = static_cast<int64_t*>(work);
                uint32_t* af = reinterpret_cast<uint32_t*>(acc + (size_t)D * F);
                k_sum_strided_sk<XSUM_DT_F64><<<num_sms, STR_WARPS * 32, STR_SMEM, s>>>(
                    static_cast<const double*>(x), outer, len, inner, o, acc, af, af + F, 1u, 0xFFFFFFFFu);
                note_launch();
                return cudaGetLastError();
            }
            e = launch_strided<XSUM_DT_F64>(x, outer, len, inner, parts, o, wk, wf, num_sms, s);
            break;
        case XSUM_DT_F32:
            e = XS_STRH ? launch_strided_f32<SF32>(x, outer, len, inner, parts, o, wk, wf, nullptr, false, num_sms, s)
                        : launch_strided<XSUM_DT_F32>(x, outer, len, inner, parts, o, wk, wf, num_sms, s);
            break;
        case XSUM_DT_F16: e = launch_strided<XSUM_DT_F16>(x, outer, len, inner, parts, o, wk, wf, num_sms, s); break;
        default: e = launch_strided<XSUM_DT_BF16>(x, outer, len, inner, parts, o, wk, wf, num_sms, s); break;
    }
    if (e != cudaSuccess || parts == 1) return e;
    if (F >= (uint64_t)num_sms * 32 * 8) {                     // many fibres: one lane each
        const unsigned gm = (unsigned)((F + STRM_WARPS * 32 - 1) / (STRM_WARPS * 32));
        k_strided_merge_lanes<<<gm, STRM_WARPS * 32, 0, s>>>(wk, wf, F, parts, o);
        note_launch();
        return cudaGetLastError();
    }
    static unsigned long long done_m = 0;
    if ((e = ensure_smem(k_strided_merge, STR_SMEM, done_m))) return e;
    const unsigned gm = (unsigned)((F + 31) / 32);
    k_strided_merge<<<gm, STR_WARPS * 32, STR_SMEM, s>>>(wk, wf, F, parts, o);
    note_launch();
    return cudaGetLastError();
}

}  // namespace xs
