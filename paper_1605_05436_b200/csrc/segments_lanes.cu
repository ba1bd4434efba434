// K11: many short equal segments (SURVEY.md §8(f) f1 "batched exact sums"): one LANE per
// segment. With one warp per segment (K6/K9), a segment of a few dozen elements still pays the
// whole warp epilogue (column combine, carry resolution, rounding: ~800 warp instructions);
// here every lane owns one segment and its private 42-digit shared-memory column (K2's lane
// column), reads the segment's elements itself and canonicalizes and rounds
// its own column (one thread; lane_round.cuh) - 32 segments per warp, no
// cross-lane step at all. The lanes of a warp read 32 consecutive segments, so a warp's loads
// cover one contiguous span of 32*len elements; loads allocate in L1, where the neighbouring
// bytes of a sector wait for the lane's next load. K11c (below) does the same for CSR segments
// that are mostly short, handing a group's longer segments to the whole warp.
#include <cuda_runtime.h>

#include "lane_round.cuh"
#include "xsum_device.cuh"
#include "xsum_kernels.h"

namespace xs {

constexpr int SL_WARPS = 16;
constexpr size_t SL_SMEM = (size_t)SL_WARPS * D * 32 * sizeof(int64_t);

// L1-allocating read-only loads (the lane revisits the rest of each sector on its next loads)
__device__ __forceinline__ uint4 ld_v4_ca(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
// Loaders: raw(p) the element's bits (L1-allocating), dec() its chunks (binary64 decompose, or
// the native narrow decode dec_narrow of lane_round.cuh), sflags() the flags of a NaN/Inf pattern.
template <int DT> struct SlLd;
template <> struct SlLd<XSUM_DT_F64> {
    using T = double;
    using R = uint2;
    __device__ static __forceinline__ R raw(const T* p) {
        uint2 v;
        asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
        return v;
    }
    __device__ static __forceinline__ Chunks dec(R r, uint32_t one) { return decompose(r.x, r.y, one); }
    __device__ static __forceinline__ uint32_t sflags(R r) { return special_flags(r.x, r.y); }
};
template <int TB, int LB>
__device__ __forceinline__ uint32_t narrow_special_flags(uint32_t b) {
    return (b & ((1u << TB) - 1)) ? XSUM_F_NAN : (((b >> (TB + LB)) & 1u) ? XSUM_F_NINF : XSUM_F_PINF);
}
template <> struct SlLd<XSUM_DT_F32> {
    using T = float;
    using R = uint32_t;
    __device__ static __forceinline__ R raw(const T* p) {
        uint32_t b;
        asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(b) : "l"(p));
        return b;
    }
    __device__ static __forceinline__ Chunks dec(R r, uint32_t) { return dec_narrow<23, 8, 925>(r); }
    __device__ static __forceinline__ uint32_t sflags(R r) { return narrow_special_flags<23, 8>(r); }
};
template <> struct SlLd<XSUM_DT_F16> {
    using T = uint16_t;
    using R = uint32_t;
    __device__ static __forceinline__ R raw(const T* p) {
        unsigned short b;
        asm volatile("ld.global.nc.b16 %0, [%1];" : "=h"(b) : "l"(p));
        return b;
    }
    __device__ static __forceinline__ Chunks dec(R r, uint32_t) { return dec_narrow<10, 5, 1050>(r); }
    __device__ static __forceinline__ uint32_t sflags(R r) { return narrow_special_flags<10, 5>(r); }
};
template <> struct SlLd<XSUM_DT_BF16> {
    using T = uint16_t;
    using R = uint32_t;
    __device__ static __forceinline__ R raw(const T* p) {
        unsigned short b;
        asm volatile("ld.global.nc.b16 %0, [%1];" : "=h"(b) : "l"(p));
        return b;
    }
    __device__ static __forceinline__ Chunks dec(R r, uint32_t) { return dec_narrow<7, 8, 941>(r); }
    __device__ static __forceinline__ uint32_t sflags(R r) { return narrow_special_flags<7, 8>(r); }
};

// Regularize digits [lo, hi] of a lane column (the only ones this segment touched; digits
// outside are zero), carrying into hi + 1; returns the new top of the touched range. Same split
// as regularize_column (balanced carry); the window's top digit is not split.
__device__ __forceinline__ int lane_regularize_range(int64_t* col, int lo, int hi) {
    int64_t cin = 0;
    const int last = hi < D - 1 ? hi : D - 2;
#pragma unroll 4
    for (int j = lo; j <= last; ++j) {
        const int64_t y = col[j * 32];
        const int64_t c = balanced_carry(y);
        col[j * 32] = y - (c << W) + cin;
        cin = c;
    }
    col[(last + 1) * 32] += cin;
    return last + 1;
}

// Round the lane's regularized column (segment s of `count` elements) into the segment outputs:
// both roundings and the flags exactly as finalize_warp reports them, and the canonical image.

__device__ __forceinline__ void lane_store_segment(int64_t* col, uint32_t flags, const SegOut& o, uint64_t s, int lo,
                                                   int hi) {
    lane_store_top(lane_canonical_top(col, lo, hi), col, flags, o, s);
}

// End of a segment in the K11 kernels (any input format): the raw digits [lo, hi] (hi < 0: nothing added)
// rounded and zeroed by one carry chain (lane_top_chain); the generic path when the image is wanted.
__device__ __forceinline__ void lane_epilogue64(int64_t* col, uint32_t flags, const SegOut& o, uint64_t s, int lo,
                                                int hi) {
    if (hi < 0) lo = hi = 0;
    if (o.canon) {
        hi = lane_regularize_range(col, lo, hi);
        lane_store_segment(col, flags, o, s, lo, hi);
#pragma unroll 4
        for (int j = lo; j <= hi; ++j) col[j * 32] = 0;
        return;
    }
    lane_store_top(lane_top_chain(col, lo, hi), col, flags, o, s);
}
#ifndef XS_SL_FAST
#define XS_SL_FAST 1
#endif
// K11s / K11 binary64: the same, trying the top-digit rounding first (lane_fast_round; values only, len <= 256)
__device__ __forceinline__ void lane_epilogue64_fast(int64_t* col, uint32_t flags, const SegOut& o, uint64_t s,
                                                     int lo, int hi, uint32_t len) {
#if XS_SL_FAST
    if (!o.canon) {
        uint64_t b64 = 0;
        uint32_t b32 = 0, rf = 0;
        if (lane_fast_round(col, lo, hi, (int64_t)len, o.out || o.flags, o.out32 || o.flags, o.flags != nullptr, b64,
                            b32, rf)) {
#pragma unroll 4
            for (int j = lo; j <= hi; ++j) col[j * 32] = 0;
            lane_store_bits(b64, b32, rf, flags, o, s);
            return;
        }
    }
#endif
    lane_epilogue64(col, flags, o, s, lo, hi);
}

template <int DT, bool VEC>
__global__ void __launch_bounds__(SL_WARPS * 32, 1)
k_segments_lanes(const typename SlLd<DT>::T* __restrict__ x, uint64_t nseg, uint64_t len, SegOut o, uint32_t one) {
    using L = SlLd<DT>;
    extern __shared__ __align__(16) int64_t win[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t* col = win + warp * (D * 32) + lane;
    const uint64_t groups = (nseg + 31) / 32;
#pragma unroll
    for (int j = 0; j < D; ++j) col[j * 32] = 0;
    for (uint64_t g = (uint64_t)blockIdx.x * SL_WARPS + warp; g < groups; g += (uint64_t)gridDim.x * SL_WARPS) {
        const uint64_t s = g * 32 + lane;
        if (s >= nseg) continue;
        uint32_t flags = 0;
#ifdef XS_SL_FULL                                    // A/B knob: always the whole column
        int lo = 0, hi = D - 1;
#else
        int lo = D, hi = -1;                         // touched digit range of this segment
#endif
        auto addr = [&](typename L::R rv) {
            Chunks c = L::dec(rv, one);
            if (spec_hit(c.spec)) { flags |= L::sflags(rv); return; }
            column_add(col, c, one);
#ifndef XS_SL_FULL
            lo = min(lo, (int)c.i);
            hi = max(hi, (int)c.i + 1);
#endif
        };
        const typename L::T* p = x + s * len;
        uint64_t r = 0;
        int since = 0;
        bool regd = false;                           // a flush regularized the column
        auto flush = [&]() {
            if (hi >= 0) hi = lane_regularize_range(col, lo, hi);
            since = 0;
            regd = true;
        };
        if (VEC) {                                   // binary64, even length, 16-B aligned rows
            const uint4* pv = reinterpret_cast<const uint4*>(p);
            for (; r + 8 <= len; r += 8) {
                uint4 v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = ld_v4_ca(pv + r / 2 + u);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if constexpr (VEC) {
                        addr(typename L::R{v[u].x, v[u].y});
                        addr(typename L::R{v[u].z, v[u].w});
                    }
                }
                since += 8;
                if (since > FLUSH_ELEMS - 8) flush();
            }
        } else {
            for (; r + 8 <= len; r += 8) {
                typename L::R v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = L::raw(p + r + u);
#pragma unroll
                for (int u = 0; u < 8; ++u) addr(v[u]);
                since += 8;
                if (since > FLUSH_ELEMS - 8) flush();
            }
        }
        for (; r < len; ++r) addr(L::raw(p + r));   // < 8 left: within the window
        if (!regd) {                                 // no regularization ran: raw digits, |y| <= len 2^52
            lane_epilogue64_fast(col, flags, o, s, lo, hi, (uint32_t)len);
            continue;
        }
        flush();
        if (hi < 0) lo = hi = 0;
        lane_store_segment(col, flags, o, s, lo, hi);
#pragma unroll 4
        for (int j = lo; j <= hi; ++j) col[j * 32] = 0;   // the rest of the column is still zero
    }
}

// K11c: CSR segments, mostly short (the caller's choice, e.g. a mean length <= 256). Warps take
// groups of 32 consecutive segments (from the ticket word in units of groups, or statically);
// every lane whose segment has <= SEG_LANES_MAX elements sums it alone as in K11 (scalar
// L1-allocating loads: CSR starts have any alignment); the group's longer segments are then
// summed one at a time by the whole warp (coalesced loads into the 32 lane columns, the raw
// column combine and finalize_warp of K6's epilogue).
template <int DT>
__global__ void __launch_bounds__(SL_WARPS * 32, 1)
k_segments_lanes_csr(const typename SlLd<DT>::T* __restrict__ x, uint64_t nseg, const uint64_t* __restrict__ offsets,
                     SegOut o, unsigned long long* __restrict__ ticket, uint32_t one) {
    using L = SlLd<DT>;
    extern __shared__ __align__(16) int64_t win[];
    __shared__ int64_t su[SL_WARPS][64];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t* col = win + warp * (D * 32) + lane;
    const uint64_t groups = (nseg + 31) / 32;
    const uint64_t nw = (uint64_t)gridDim.x * SL_WARPS;
#pragma unroll
    for (int j = 0; j < D; ++j) col[j * 32] = 0;
    uint64_t g = ticket ? seg_next(ticket, 0, nw, lane) : (uint64_t)blockIdx.x * SL_WARPS + warp;
    while (g < groups) {
        const uint64_t gn = seg_next(ticket, g, nw, lane);        // next group, drawn early
        const uint64_t s = g * 32 + lane;
        const bool act = s < nseg;
        const uint64_t b = act ? __ldg(offsets + s) : 0, e = act ? __ldg(offsets + s + 1) : 0;
        const uint64_t len = e - b;
        const bool small = act && len <= SEG_LANES_MAX;
        if (small) {                                             // one lane, one segment
            uint32_t flags = 0;
            int lo = D, hi = -1;
            auto addr = [&](typename L::R rv) {
                Chunks c = L::dec(rv, one);
                if (spec_hit(c.spec)) { flags |= L::sflags(rv); return; }
                column_add(col, c, one);
                lo = min(lo, (int)c.i);
                hi = max(hi, (int)c.i + 1);
            };
            const typename L::T* p = x + b;
            uint64_t r = 0;
            for (; r + 8 <= len; r += 8) {                       // len <= 256 < FLUSH_ELEMS: one window
                typename L::R v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = L::raw(p + r + u);
#pragma unroll
                for (int u = 0; u < 8; ++u) addr(v[u]);
            }
            for (; r < len; ++r) addr(L::raw(p + r));
            lane_epilogue64_fast(col, flags, o, s, lo, hi, (uint32_t)len);   // raw digits (<= 256 adds)
        }
        unsigned long long big = __ballot_sync(FULL, act && !small);
        while (big) {                                            // long segments: the whole warp
            const int j = __ffsll((long long)big) - 1;
            big &= big - 1;
            const uint64_t bj = __shfl_sync(FULL, b, j), ej = __shfl_sync(FULL, e, j);
            uint32_t flags = 0;
            int since = 0;
            uint64_t r = bj + lane;
            for (; r + 7 * 32 < ej; r += 8 * 32) {
                typename L::R v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = L::raw(x + r + u * 32);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    Chunks c = L::dec(v[u], one);
                    if (spec_hit(c.spec)) flags |= L::sflags(v[u]);
                    else column_add(col, c, one);
                }
                since += 8;
                if (since > FLUSH_ELEMS - 8) {
                    regularize_column(col);
                    since = 0;
                }
            }
            for (; r < ej; r += 32) {                            // < 8 per lane left: in the window
                const typename L::R v = L::raw(x + r);
                Chunks c = L::dec(v, one);
                if (spec_hit(c.spec)) flags |= L::sflags(v);
                else column_add(col, c, one);
            }
            __syncwarp();
            int64_t a0, a1;
            combine_raw_columns(win + warp * (D * 32), a0, a1, lane);
            __syncwarp();
#pragma unroll
            for (int d = 0; d < D; ++d) col[d * 32] = 0;
            const uint32_t fl = __reduce_or_sync(FULL, flags);
            const uint64_t sj = g * 32 + j;
            xsum_result res = finalize_warp(a0, a1, fl, ej - bj, o.canon ? o.canon + sj * XSUM_CANON_LIMBS : nullptr,
                                            su[warp], lane);
            if (lane == 0) o.write(sj, res);
        }
        g = gn;
    }
}

template <int DT>
static cudaError_t launch_lanes_csr(const void* x, uint64_t nseg, const uint64_t* offsets, const SegOut& o,
                                    unsigned long long* ticket, int num_sms, cudaStream_t s) {
    static unsigned long long done = 0;
    if (cudaError_t e = ensure_smem(k_segments_lanes_csr<DT>, SL_SMEM, done)) return e;
    const uint64_t groups = (nseg + 31) / 32;
    const uint64_t want = (groups + SL_WARPS - 1) / SL_WARPS;
    const unsigned g = (unsigned)(want < (uint64_t)num_sms ? want : num_sms);
    k_segments_lanes_csr<DT><<<g, SL_WARPS * 32, SL_SMEM, s>>>(static_cast<const typename SlLd<DT>::T*>(x), nseg,
                                                               offsets, o, ticket, 1u);
    note_launch();
    return cudaGetLastError();
}

cudaError_t sum_segments_lanes_csr(const void* x, int dtype, uint64_t nseg, const uint64_t* offsets, const SegOut& o,
                                   unsigned long long* ticket, int num_sms, cudaStream_t s) {
    if (nseg == 0) return cudaSuccess;
    switch (dtype) {
        case XSUM_DT_F64: return launch_lanes_csr<XSUM_DT_F64>(x, nseg, offsets, o, ticket, num_sms, s);
        case XSUM_DT_F32: return launch_lanes_csr<XSUM_DT_F32>(x, nseg, offsets, o, ticket, num_sms, s);
        case XSUM_DT_F16: return launch_lanes_csr<XSUM_DT_F16>(x, nseg, offsets, o, ticket, num_sms, s);
        default: return launch_lanes_csr<XSUM_DT_BF16>(x, nseg, offsets, o, ticket, num_sms, s);
    }
}

// K11 for binary64 rows that are 16-B aligned with an even length <= SEG_LANES_MAX (c5s16): the
// next segment's first SLP elements are loaded before this segment is summed and rounded, so they
// are in flight through its adds and epilogue (the per-segment epilogue otherwise leaves the load
// pipe idle: ncu r01, 26% of stall samples on the first use of a load); NaN/Inf patterns are summed
// unchecked like finite values and, if the lane saw one, cancelled by a rescan of its segment
// (K2's scheme; <= 2 x 256 adds stay far inside the int64 headroom, so no flush is needed).
constexpr int SLP = 16;                     // elements prefetched per lane (8 x 16 B)
#ifndef XS_SL_PF
#define XS_SL_PF 1
#endif
#ifndef XS_SL_TMA
#define XS_SL_TMA 1          // short rows through the bulk-copy staging kernel (k_segments_lanes64s)
#endif
__global__ void __launch_bounds__(SL_WARPS * 32, 1)
k_segments_lanes64(const double* __restrict__ x, uint64_t nseg, uint64_t len, SegOut o, uint32_t one, uint32_t mone) {
    extern __shared__ __align__(16) int64_t win[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t* col = win + warp * (D * 32) + lane;
    const uint64_t groups = (nseg + 31) / 32;
#pragma unroll
    for (int j = 0; j < D; ++j) col[j * 32] = 0;
    const uint64_t gstride = (uint64_t)gridDim.x * SL_WARPS;
    const int npf = (int)(len < (uint64_t)SLP ? len : (uint64_t)SLP) / 2;     // vectors prefetched
    uint4 pf[SLP / 2];
    auto prefetch = [&](uint64_t gg) {
        const uint64_t s = gg * 32 + lane;
        if (gg < groups && s < nseg) {
            const uint4* pv = reinterpret_cast<const uint4*>(x + s * len);
#pragma unroll
            for (int u = 0; u < SLP / 2; ++u)
                if (u < npf) pf[u] = ld_v4_ca(pv + u);
        }
    };
    uint64_t g = (uint64_t)blockIdx.x * SL_WARPS + warp;
    prefetch(g);
    for (; g < groups; g += gstride) {
        const uint64_t s = g * 32 + lane;
        uint4 cur[SLP / 2];
#pragma unroll
        for (int u = 0; u < SLP / 2; ++u) cur[u] = pf[u];
#if XS_SL_PF
        prefetch(g + gstride);
#endif
        if (s >= nseg) continue;
        // the segment's exponent band in one packed 16x2 max (lo16: max k, hi16: 0xFFFF - min k; K6z)
        uint32_t band = 0, flags = 0;
        auto addc = [&](uint32_t xl, uint32_t xh) {
            const Chunks c = decompose(xl, xh, one, mone);
            column_add(col, c, one);
            band = __vmaxu2(band, mad_u32(c.spec, 0xFFFF0001u, 0xFFFF0000u));
        };
#if !XS_SL_PF
        {
            const uint4* pv0 = reinterpret_cast<const uint4*>(x + s * len);
#pragma unroll
            for (int u = 0; u < SLP / 2; ++u)
                if (u < npf) cur[u] = ld_v4_ca(pv0 + u);
        }
#endif
#pragma unroll
        for (int u = 0; u < SLP / 2; ++u) {
            if (u < npf) {
                addc(cur[u].x, cur[u].y);
                addc(cur[u].z, cur[u].w);
            }
        }
        const uint4* pv = reinterpret_cast<const uint4*>(x + s * len);
        uint64_t r = 2 * (uint64_t)npf;
        for (; r + 8 <= len; r += 8) {
            uint4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = ld_v4_ca(pv + r / 2 + u);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                addc(v[u].x, v[u].y);
                addc(v[u].z, v[u].w);
            }
        }
        for (; r < len; r += 2) {
            const uint4 v = ld_v4_ca(pv + r / 2);
            addc(v.x, v.y);
            addc(v.z, v.w);
        }
        const int lo = (0xFFFF - (int)(band >> 16)) / 52, hi = (int)(band & 0xFFFFu) / 52 + 1;
        if (spec_hit(band & 0xFFFFu)) {               // rare: cancel the NaN/Inf patterns (R10)
            for (uint64_t q = 0; q < len; q += 2) {
                const uint4 v = ld_v4_ca(pv + q / 2);
                column_fix_special(col, v.x, v.y, flags, one);
                column_fix_special(col, v.z, v.w, flags, one);
            }
        }
        lane_epilogue64_fast(col, flags, o, s, lo, hi, (uint32_t)len);
    }
}

// K11 for SHORT binary64 rows (even length <= SLS_MAX, 16-B aligned; c5s16): a warp's 32 segments are
// one contiguous span of 32 * len doubles, fetched by ONE bulk copy (cp.async.bulk, the TMA engine)
// into a shared-memory staging buffer - double-buffered per warp, the next group's copy in flight
// while this group is summed - and each lane reads its own segment from shared memory, in a
// rotated vector order that keeps a quarter warp on distinct banks (the sum is order-free). The
// per-lane 16-B global loads of k_segments_lanes64 touch 32 lines per warp instruction: ncu (r02)
// showed the L1 data pipe 84% busy, half of it global-load wavefronts.
#ifndef XS_SLS_NBUF
#define XS_SLS_NBUF 1            // staging buffers per warp (tools/variants.py: 1 -> 15 warps, 2 -> 12 warps)
#endif
constexpr int SLS_NBUF = XS_SLS_NBUF;
// lane columns 10.5 KB + NBUF x 4 KB staging per warp: 15 x 14.5 KB / 12 x 18.5 KB <= 227 KB
constexpr int SLS_WARPS = SLS_NBUF == 1 ? 15 : 12;
constexpr int SLS_MAX = 16;                    // doubles per segment (4 KB per group of 32 segments)
constexpr size_t SLS_STAGE = 32 * SLS_MAX * 8;
constexpr size_t SLS_SMEM = (size_t)SLS_WARPS * (D * 32 * 8 + SLS_NBUF * SLS_STAGE) + SLS_WARPS * 2 * 8;

__device__ __forceinline__ void mbar_init(uint32_t bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(bar), "r"(phase) : "memory");
    }
}

__global__ void __launch_bounds__(SLS_WARPS * 32, 1)
k_segments_lanes64s(const double* __restrict__ x, uint64_t nseg, uint32_t len, SegOut o, uint32_t one, uint32_t mone) {
    extern __shared__ __align__(16) int64_t win[];   // bulk copies need 16-B aligned destinations
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t* col = win + warp * (D * 32) + lane;
    uint8_t* stage = reinterpret_cast<uint8_t*>(win + SLS_WARPS * D * 32) + (size_t)warp * SLS_NBUF * SLS_STAGE;
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(win + SLS_WARPS * D * 32) +
                                                 (size_t)SLS_WARPS * SLS_NBUF * SLS_STAGE) + warp * 2;
    const uint32_t stage_s = (uint32_t)__cvta_generic_to_shared(stage);
    const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(bars);
    const uint64_t groups = (nseg + 31) / 32;
    const uint64_t gstride = (uint64_t)gridDim.x * SLS_WARPS;
    const uint32_t nv = len / 2;                                 // 16-B vectors per segment
#pragma unroll
    for (int j = 0; j < D; ++j) col[j * 32] = 0;
    if (lane == 0) {
        mbar_init(bar_s);
        mbar_init(bar_s + 8);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    auto issue = [&](uint64_t gg, int b) {
        if (lane == 0 && gg < groups) {
            const uint64_t s0 = gg * 32;
            const uint64_t ns = nseg - s0 < 32 ? nseg - s0 : 32;
            bulk_load(stage_s + b * (uint32_t)SLS_STAGE, x + s0 * len, (uint32_t)(ns * len * 8), bar_s + 8 * b);
        }
    };
    uint64_t g = (uint64_t)blockIdx.x * SLS_WARPS + warp;
    issue(g, 0);
    uint32_t phases = 0;                                         // bit b: the parity buffer b waits for
    int b = 0;
    for (; g < groups; g += gstride) {
        if (SLS_NBUF == 2) issue(g + gstride, b ^ 1);            // in flight while this group is summed
        mbar_wait(bar_s + 8 * b, (phases >> b) & 1u);
        phases ^= 1u << b;
        const uint64_t s = g * 32 + lane;
        const bool mine = s < nseg;
        int lo = D, hi = -1;
        uint32_t flags = 0;
        if (mine) {
            const uint4* sv = reinterpret_cast<const uint4*>(stage + b * SLS_STAGE + (size_t)lane * len * 8);
            // the exponent band of the segment in ONE packed 16x2 max per two summands (lo16: max k,
            // also the NaN/Inf detector; hi16: 0xFFFF - min k), as K6z: chunks land in digits
            // [k_min / 52, k_max / 52 + 1]
            uint32_t band = 0;
            auto key = [&](const Chunks& c) { return mad_u32(c.spec, 0xFFFF0001u, 0xFFFF0000u); };
            uint32_t u = (uint32_t)lane % nv;                    // rotated start: distinct banks
#pragma unroll 4
            for (uint32_t q = 0; q < nv; ++q) {
                const uint4 v = sv[u];
                const Chunks ca = decompose(v.x, v.y, one, mone);
                column_add(col, ca, one);
                const Chunks cb = decompose(v.z, v.w, one, mone);
                column_add(col, cb, one);
                band = __vmaxu2(__vmaxu2(band, key(ca)), key(cb));
                u = u + 1 == nv ? 0 : u + 1;
            }
            const int kmax = (int)(band & 0xFFFFu), kmin = 0xFFFF - (int)(band >> 16);
            lo = kmin / 52;
            hi = kmax / 52 + 1;
            if (spec_hit((uint32_t)kmax)) {                      // rare: cancel NaN/Inf patterns (R10)
                for (uint32_t q = 0; q < nv; ++q) {
                    const uint4 v = sv[q];
                    column_fix_special(col, v.x, v.y, flags, one);
                    column_fix_special(col, v.z, v.w, flags, one);
                }
            }
        }
        __syncwarp();                                            // this group's staging is consumed
        if (SLS_NBUF == 1) issue(g + gstride, 0);                // the next copy overlaps the epilogue
        if (mine) lane_epilogue64_fast(col, flags, o, s, lo, hi, len);
        if (SLS_NBUF == 2) b ^= 1;
    }
}

static cudaError_t launch_lanes64s(const void* x, uint64_t nseg, uint64_t len, const SegOut& o, int num_sms,
                                   cudaStream_t s) {
    static unsigned long long done = 0;
    if (cudaError_t e = ensure_smem(k_segments_lanes64s, SLS_SMEM, done)) return e;
    const uint64_t groups = (nseg + 31) / 32;
    const uint64_t want = (groups + SLS_WARPS - 1) / SLS_WARPS;
    const unsigned g = (unsigned)(want < (uint64_t)num_sms ? want : num_sms);
    k_segments_lanes64s<<<g, SLS_WARPS * 32, SLS_SMEM, s>>>(static_cast<const double*>(x), nseg, (uint32_t)len, o, 1u,
                                                            0xFFFFFFFFu);
    note_launch();
    return cudaGetLastError();
}

static cudaError_t launch_lanes64(const void* x, uint64_t nseg, uint64_t len, const SegOut& o, int num_sms,
                                  cudaStream_t s) {
    static unsigned long long done = 0;
    if (cudaError_t e = ensure_smem(k_segments_lanes64, SL_SMEM, done)) return e;
    const uint64_t groups = (nseg + 31) / 32;
    const uint64_t want = (groups + SL_WARPS - 1) / SL_WARPS;
    const unsigned g = (unsigned)(want < (uint64_t)num_sms ? want : num_sms);
    k_segments_lanes64<<<g, SL_WARPS * 32, SL_SMEM, s>>>(static_cast<const double*>(x), nseg, len, o, 1u,
                                                         0xFFFFFFFFu);
    note_launch();
    return cudaGetLastError();
}

template <int DT, bool VEC>
static cudaError_t launch_lanes(const void* x, uint64_t nseg, uint64_t len, const SegOut& o, int num_sms,
                                cudaStream_t s) {
    static unsigned long long done = 0;
    if (cudaError_t e = ensure_smem(k_segments_lanes<DT, VEC>, SL_SMEM, done)) return e;
    const uint64_t groups = (nseg + 31) / 32;
    const uint64_t want = (groups + SL_WARPS - 1) / SL_WARPS;
    const unsigned g = (unsigned)(want < (uint64_t)num_sms ? want : num_sms);
    k_segments_lanes<DT, VEC><<<g, SL_WARPS * 32, SL_SMEM, s>>>(static_cast<const typename SlLd<DT>::T*>(x), nseg,
                                                                len, o, 1u);
    note_launch();
    return cudaGetLastError();
}

cudaError_t sum_segments_lanes(const void* x, int dtype, uint64_t nseg, uint64_t len, const SegOut& o, int num_sms,
                               cudaStream_t s) {
    if (nseg == 0) return cudaSuccess;
    switch (dtype) {
        case XSUM_DT_F64:
            if (len % 2 == 0 && ((uintptr_t)x & 15) == 0)
                return len <= (uint64_t)SLS_MAX && XS_SL_TMA ? launch_lanes64s(x, nseg, len, o, num_sms, s)
                       : len <= SEG_LANES_MAX ? launch_lanes64(x, nseg, len, o, num_sms, s)
                                              : launch_lanes<XSUM_DT_F64, true>(x, nseg, len, o, num_sms, s);
            return launch_lanes<XSUM_DT_F64, false>(x, nseg, len, o, num_sms, s);
        case XSUM_DT_F32: return launch_lanes<XSUM_DT_F32, false>(x, nseg, len, o, num_sms, s);
        case XSUM_DT_F16: return launch_lanes<XSUM_DT_F16, false>(x, nseg, len, o, num_sms, s);
        default: return launch_lanes<XSUM_DT_BF16, false>(x, nseg, len, o, num_sms, s);
    }
}

}  // namespace xs
