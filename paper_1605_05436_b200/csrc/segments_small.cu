// K9: segmented exact sums of binary32 / binary16 / bfloat16 elements (SURVEY.md §8(f) f1 x f2:
// reproducible reductions of the formats tensors are usually stored in).
//
// One warp per segment (the paper's per-partition combine), lanes striding
// over the segment with 16-byte loads. Each element of the paper's t-bit / l-bit format
// is M 2^k in units of its least subnormal (M < 2^(t+1), k = max(e,1) - 1),
// i.e. M at bit k + OFF of the 2^-1074 window (binary32 OFF = 925, binary16 1050, bfloat16 941).
// As in K8, each lane adds M 2^(ep mod 32) (ep = max(e,1)) into an unsigned 64-bit bin per
// (sign, group of 32 exponents) - one 64-bit read-modify-write per element, carries deferred
// - and empties the bins into a narrow digit column (only the digits the
// format reaches, from COL0 on) every 511 adds and at the segment's end. NaN/Inf patterns are
// summed as if finite; a per-lane max of ep sends a segment that held one to a rescan that
// cancels them exactly and sets the flags (reading R10). At the segment's end the 32 narrow
// columns are combined, moved to their digit positions and rounded by finalize_warp (binary64
// and binary32). CSR segments are drawn from a ticket word as in K6; equal
// segments of <= SEG_LANES_MAX elements go to K11 (one lane per segment).
#include <cuda_runtime.h>

#include "f32_bins.cuh"
#include "h16_common.cuh"
#include "lane_round.cuh"
#include "xsum_device.cuh"
#include "xsum_kernels.h"

namespace xs {

template <class F>
__device__ __forceinline__ uint32_t sload_one(const uint8_t* p) {
    if (F::eb == 4) return __ldg(reinterpret_cast<const uint32_t*>(p));
    return __ldg(reinterpret_cast<const uint16_t*>(p));
}

#ifndef XS_SSEG_WARPS
#define XS_SSEG_WARPS 16   // one 16-warp block per SM: segments of 4096 binary32 1030 -> 1100, binary16 1949 -> 2011-2039, bfloat16 1655 -> 1676 G/s
#endif
#ifndef XS_SSEG_MINB
#define XS_SSEG_MINB 1
#endif
constexpr int SSEG_WARPS = XS_SSEG_WARPS;
constexpr int SSEG_U = 4;                  // vectors per lane per tile

template <class F>
constexpr size_t sseg_smem() { return (size_t)SSEG_WARPS * 32 * (F::COLS + F::NBIN) * sizeof(int64_t); }

// Rare path: the segment held NaN/Inf patterns (summed as finite values): re-read it, set the
// flags and cancel them (the sign-flipped pattern lands in the other sign's bin of the same
// group), flush.
template <class F>
__device__ __noinline__ void sseg_rescan(uint64_t* bins, int64_t* col, const uint8_t* xs, uint64_t head,
                                         const uint4* body, uint64_t nvec, uint64_t tail, int lane, uint32_t& flags,
                                         uint32_t one) {
    uint32_t dummy = 0, adds = 0, flushes = 0;
    scol_regularize<F>(col);                            // fresh headroom for the flushes below
    auto fix = [&](uint32_t b) {
        const uint32_t f = sspecial_flags<F>(b);
        if (f) {
            flags |= f;
            sbin_add<F>(bins, b ^ (1u << (F::t + F::l)), dummy, one);
            if (++adds == SSEG_FLUSH) {                 // a lane may cancel any number of specials
                sbin_flush<F>(bins, col);
                adds = 0;
                if (++flushes == SSEG_REG_FLUSHES) { scol_regularize<F>(col); flushes = 0; }
            }
        }
    };
    if ((uint64_t)lane < head) fix(sload_one<F>(xs + lane * F::eb));
    if (lane >= 8 && (uint64_t)(lane - 8) < tail) fix(sload_one<F>(xs + (head + nvec * F::per_vec + (lane - 8)) * F::eb));
    for (uint64_t v = lane; v < nvec; v += 32) {
        const uint4 q = ldg_stream(body + v);
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
        for (int i = 0; i < 4; ++i) {
            if (F::eb == 4) {
                fix(w[i]);
            } else {
                fix(w[i] & 0xFFFFu);
                fix(w[i] >> 16);
            }
        }
    }
    sbin_flush<F>(bins, col);
}

template <class F>
__global__ void __launch_bounds__(SSEG_WARPS * 32, XS_SSEG_MINB)
k_segments_small(const uint8_t* __restrict__ x, uint64_t nseg, uint64_t seg_len, const uint64_t* __restrict__ offsets,
                 SegOut o, unsigned long long* __restrict__ ticket, uint32_t one) {
    extern __shared__ __align__(16) int64_t win[];
    __shared__ int64_t su[SSEG_WARPS][64];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t* col = win + warp * (F::COLS * 32) + lane;
    const int64_t* wb = win + warp * (F::COLS * 32);
    uint64_t* bins = reinterpret_cast<uint64_t*>(win + SSEG_WARPS * F::COLS * 32) + warp * (F::NBIN * 32) + lane;
    const uint64_t nw = (uint64_t)gridDim.x * SSEG_WARPS;
    constexpr int PV = F::per_vec;
    constexpr int SU = SSEG_U;
    constexpr uint32_t WIN_TILES = (SSEG_FLUSH - 2 - SU * PV) / (SU * PV);   // + leftovers + head/tail
    struct Seg {
        const uint8_t* xs;
        uint64_t len, head, nvec, tail, nit;
        const uint4* body;
    };
    auto open_seg = [&](uint64_t sj) {
        Seg g;
        const uint64_t beg = offsets ? offsets[sj] : sj * seg_len;
        g.len = offsets ? offsets[sj + 1] - beg : seg_len;
        g.xs = x + beg * F::eb;
        g.head = ((16 - ((uintptr_t)g.xs & 15)) & 15) / F::eb;
        if (g.head > g.len) g.head = g.len;
        g.nvec = (g.len - g.head) / PV;
        g.tail = g.len - g.head - g.nvec * PV;
        g.body = reinterpret_cast<const uint4*>(g.xs + g.head * F::eb);
        g.nit = g.nvec / (32 * SU);
        return g;
    };
    uint64_t s = ticket ? seg_next(ticket, 0, nw, lane) : (uint64_t)blockIdx.x * SSEG_WARPS + warp;
    if (s >= nseg) return;                                  // warp-uniform
#pragma unroll
    for (int j = 0; j < F::COLS; ++j) col[j * 32] = 0;
#pragma unroll
    for (int j = 0; j < F::NBIN; ++j) bins[j * 32] = 0;
    Seg g = open_seg(s);
    uint4 cur[SU], alt[SU];
    if (g.nit) {
#pragma unroll
        for (int u = 0; u < SU; ++u) cur[u] = ldg_stream(g.body + u * 32 + lane);
    }
    while (true) {
        const uint64_t sn = seg_next(ticket, s, nw, lane);     // drawn early: its latency hides
        uint32_t flags = 0, since = 0, spec = 0, flushes = 0;
        const uint64_t nit = g.nit, nvec = g.nvec;
        const uint4* body = g.body;
        // head / tail: one element per lane (head < PV <= 8, tail < PV)
        if ((uint64_t)lane < g.head) sbin_add<F>(bins, sload_one<F>(g.xs + lane * F::eb), spec, one);
        if (lane >= 8 && (uint64_t)(lane - 8) < g.tail)
            sbin_add<F>(bins, sload_one<F>(g.xs + (g.head + nvec * PV + (lane - 8)) * F::eb), spec, one);
        // full tiles: two register buffers alternate (tile it+1 loads while tile it is added)
        auto process = [&](const uint4 (&bf)[SU]) {
#pragma unroll
            for (int u = 0; u < SU; ++u) sbin_add_vec<F>(bins, bf[u], spec, one);
            if (++since == WIN_TILES) {
                sbin_flush<F>(bins, col);
                since = 0;
                if (++flushes == SSEG_REG_FLUSHES) { scol_regularize<F>(col); flushes = 0; }
            }
        };
        for (uint64_t it = 0; it < nit; it += 2) {
            if (it + 1 < nit) {
#pragma unroll
                for (int u = 0; u < SU; ++u) alt[u] = ldg_stream(body + (it + 1) * (32 * SU) + u * 32 + lane);
            }
            process(cur);
            if (it + 1 >= nit) break;
            if (it + 2 < nit) {
#pragma unroll
                for (int u = 0; u < SU; ++u) cur[u] = ldg_stream(body + (it + 2) * (32 * SU) + u * 32 + lane);
            }
            process(alt);
        }
        // leftover vectors (< one tile), loaded together before use
        uint4 lv[SU];
#pragma unroll
        for (int u = 0; u < SU; ++u) {
            const uint64_t v = nit * (32 * SU) + u * 32 + lane;
            if (v < nvec) lv[u] = ldg_stream(body + v);
        }
#pragma unroll
        for (int u = 0; u < SU; ++u)
            if (nit * (32 * SU) + u * 32 + lane < nvec) sbin_add_vec<F>(bins, lv[u], spec, one);
        sbin_flush<F>(bins, col);
        if (__any_sync(FULL, spec == F::EM))            // rare: NaN/Inf patterns in this segment
            sseg_rescan<F>(bins, col, g.xs, g.head, body, nvec, g.tail, lane, flags, one);
        // prefetch the next segment, then close this one
        const bool more = sn < nseg;
        const uint64_t len = g.len;
        if (more) {
            g = open_seg(sn);
            if (g.nit) {
#pragma unroll
                for (int u = 0; u < SU; ++u) cur[u] = ldg_stream(g.body + u * 32 + lane);
            }
        }
        // combine: lane r < COLS sums row r over the 32 lanes (hi/lo halves: raw |Y| < 2^63),
        // splits balanced carries (the top row is not split), the carries move one row up, and
        // the rows move to their digit positions
        __syncwarp();
        int64_t hs = 0, ls = 0;
        if (lane < F::COLS) {
#pragma unroll 8
            for (int c = 0; c < 32; ++c) {
                const int64_t v = wb[lane * 32 + ((lane + c) & 31)];
                hs += v >> 32;
                ls += (int64_t)(uint32_t)v;
            }
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < F::COLS; ++j) col[j * 32] = 0;
        int64_t cr = 0, rr = (int64_t)((uint64_t)hs << 32) + ls;
        if (lane < F::COLS - 1) {
            cr = (hs + ((ls + (1ll << 51)) >> 32)) >> 20;
            rr = (int64_t)((uint64_t)(hs - (cr << 20)) << 32) + ls;
        }
        int64_t cin = __shfl_up_sync(FULL, cr, 1);
        if (lane == 0) cin = 0;
        const int64_t row = lane < F::COLS ? rr + cin : 0;
        const int64_t d = __shfl_sync(FULL, row, (lane - F::COL0) & 31);
        const int64_t a0 = (lane >= F::COL0 && lane < F::COL0 + F::COLS) ? d : 0;
        flags = __reduce_or_sync(FULL, flags);
        const xsum_result r =
            finalize_warp_inl(a0, 0, flags, len, o.canon ? o.canon + s * XSUM_CANON_LIMBS : nullptr, su[warp], lane);
        if (lane == 0) o.write(s, r);
        __syncwarp();
        if (!more) break;
        s = sn;
    }
}

// ---------------------------------------------------------------------------------------
// 16-bit formats: the decode and bins of K7 (h16_common.cuh: both halves of a word decoded in
// 16-bit lanes, unsigned 32-bit bins per (sign, group of 2^SB exponents) fed by fire-and-forget
// red.shared, NaN/Inf in a group of their own that is never summed) with a per-segment flush
// into a narrow digit column. About 11 instructions per element instead of ~17.
// ---------------------------------------------------------------------------------------
// Rare path: classify the NaN/Inf patterns of a segment (they were binned into the special
// group, which is never summed).
template <class F>
__device__ __noinline__ uint32_t h16seg_classify(const uint16_t* xs, uint64_t len, int lane) {
    uint32_t f = 0;
    for (uint64_t i = lane; i < len; i += 32) f |= h16_special_flags<F>(__ldg(xs + i));
    return f;
}

template <class F>
__device__ __forceinline__ void h16seg_add_checked(uint32_t* bins, uint32_t b16, uint32_t& flags) {
    const uint32_t f = h16_special_flags<F>(b16);
    if (f) { flags |= f; return; }
    h16_add<F>(bins, b16 & 0x7FFFu, b16 >> 15);
}

template <class F>
constexpr size_t h16seg_smem() {
    return (size_t)SSEG_WARPS * 32 * (H16Col<F>::COLS * 8 + F::NBIN * 4);
}

template <class F>
__global__ void __launch_bounds__(SSEG_WARPS * 32, XS_SSEG_MINB)
k_segments_h16(const uint16_t* __restrict__ x, uint64_t nseg, uint64_t seg_len, const uint64_t* __restrict__ offsets,
               SegOut o, unsigned long long* __restrict__ ticket, uint32_t one, uint32_t mone) {
    using S = H16Col<F>;
    extern __shared__ __align__(16) int64_t win[];
    __shared__ int64_t su[SSEG_WARPS][64];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t* col = win + warp * (S::COLS * 32) + lane;
    const int64_t* wb = win + warp * (S::COLS * 32);
    uint32_t* bins = reinterpret_cast<uint32_t*>(win + SSEG_WARPS * S::COLS * 32) + warp * (F::NBIN * 32) + lane;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(bins);
    const uint32_t sbase2 = sbase * 0x00010001u;
    const uint64_t nw = (uint64_t)gridDim.x * SSEG_WARPS;
    constexpr int PV = 8;
    constexpr int SU = SSEG_U;
    constexpr uint32_t WIN_TILES = (F::FLUSH - 2 - SU * PV) / (SU * PV);   // + leftovers + head/tail
    static_assert(WIN_TILES >= 1, "window shorter than one tile");
    struct Seg {
        const uint16_t* xs;
        uint64_t len, head, nvec, tail, nit;
        const uint4* body;
    };
    auto open_seg = [&](uint64_t sj) {
        Seg g;
        const uint64_t beg = offsets ? offsets[sj] : sj * seg_len;
        g.len = offsets ? offsets[sj + 1] - beg : seg_len;
        g.xs = x + beg;
        g.head = ((16 - ((uintptr_t)g.xs & 15)) & 15) / 2;
        if (g.head > g.len) g.head = g.len;
        g.nvec = (g.len - g.head) / PV;
        g.tail = g.len - g.head - g.nvec * PV;
        g.body = reinterpret_cast<const uint4*>(g.xs + g.head);
        g.nit = g.nvec / (32 * SU);
        return g;
    };
    uint64_t s = ticket ? seg_next(ticket, 0, nw, lane) : (uint64_t)blockIdx.x * SSEG_WARPS + warp;
    if (s >= nseg) return;                                  // warp-uniform
#pragma unroll
    for (int j = 0; j < S::COLS; ++j) col[j * 32] = 0;
#pragma unroll
    for (int j = 0; j < F::NBIN; ++j) bins[j * 32] = 0;
    Seg g = open_seg(s);
    uint4 cur[SU], alt[SU];
    if (g.nit) {
#pragma unroll
        for (int u = 0; u < SU; ++u) cur[u] = ldg_stream(g.body + u * 32 + lane);
    }
    while (true) {
        const uint64_t sn = seg_next(ticket, s, nw, lane);     // drawn early: its latency hides
        uint32_t flags = 0, since = 0, flushes = 0;
        bool special = false;
        const uint64_t nit = g.nit, nvec = g.nvec;
        const uint4* body = g.body;
        if ((uint64_t)lane < g.head) h16seg_add_checked<F>(bins, __ldg(g.xs + lane), flags);
        if (lane >= 8 && (uint64_t)(lane - 8) < g.tail)
            h16seg_add_checked<F>(bins, __ldg(g.xs + g.head + nvec * PV + (lane - 8)), flags);
        auto process = [&](const uint4 (&bf)[SU]) {
#pragma unroll
            for (int u = 0; u < SU; ++u) {
                h16_add_word<F>(sbase, sbase2, bf[u].x, one, mone);
                h16_add_word<F>(sbase, sbase2, bf[u].y, one, mone);
                h16_add_word<F>(sbase, sbase2, bf[u].z, one, mone);
                h16_add_word<F>(sbase, sbase2, bf[u].w, one, mone);
            }
            if (++since == WIN_TILES) {
                special |= h16_flush_col<F>(bins, col);
                since = 0;
                if (++flushes == S::REG_FLUSHES) { h16_col_regularize<F>(col); flushes = 0; }
            }
        };
        for (uint64_t it = 0; it < nit; it += 2) {
            if (it + 1 < nit) {
#pragma unroll
                for (int u = 0; u < SU; ++u) alt[u] = ldg_stream(body + (it + 1) * (32 * SU) + u * 32 + lane);
            }
            process(cur);
            if (it + 1 >= nit) break;
            if (it + 2 < nit) {
#pragma unroll
                for (int u = 0; u < SU; ++u) cur[u] = ldg_stream(body + (it + 2) * (32 * SU) + u * 32 + lane);
            }
            process(alt);
        }
        uint4 lv[SU];
#pragma unroll
        for (int u = 0; u < SU; ++u) {
            const uint64_t v = nit * (32 * SU) + u * 32 + lane;
            if (v < nvec) lv[u] = ldg_stream(body + v);
        }
#pragma unroll
        for (int u = 0; u < SU; ++u) {
            if (nit * (32 * SU) + u * 32 + lane < nvec) {
                h16_add_word<F>(sbase, sbase2, lv[u].x, one, mone);
                h16_add_word<F>(sbase, sbase2, lv[u].y, one, mone);
                h16_add_word<F>(sbase, sbase2, lv[u].z, one, mone);
                h16_add_word<F>(sbase, sbase2, lv[u].w, one, mone);
            }
        }
        special |= h16_flush_col<F>(bins, col);
        if (__any_sync(FULL, special)) flags |= h16seg_classify<F>(g.xs, g.len, lane);   // rare
        const bool more = sn < nseg;
        const uint64_t len = g.len;
        if (more) {
            g = open_seg(sn);
            if (g.nit) {
#pragma unroll
                for (int u = 0; u < SU; ++u) cur[u] = ldg_stream(g.body + u * 32 + lane);
            }
        }
        __syncwarp();
        const int64_t a0 = h16_col_combine<F>(wb, lane);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < S::COLS; ++j) col[j * 32] = 0;
        flags = __reduce_or_sync(FULL, flags);
        const xsum_result r =
            finalize_warp_inl(a0, 0, flags, len, o.canon ? o.canon + s * XSUM_CANON_LIMBS : nullptr, su[warp], lane);
        if (lane == 0) o.write(s, r);
        __syncwarp();
        if (!more) break;
        s = sn;
    }
}

// ---------------------------------------------------------------------------------------
// Equal 16-bit segments (16-B aligned, length a multiple of 8): a QUARTER warp per segment, four
// segments per warp at a time. The whole-warp kernel pays its epilogue (bins -> column, the
// combine of 32 lane columns, finalize_warp: ~550 warp instructions) for every 4096-element
// (8 KB) segment - 44% of its instructions (ncu r02: issue 74%, ALU 75%). Here the 8 lanes of a
// group stream their segment (128 B per load instruction, coalesced), empty their bins into their
// narrow columns, sum the group's 8 columns row by row into a shared row vector (raw digits), and
// ONE lane rounds it with the carry chain of K11 (lane_top_chain) - the four groups' leaders in
// parallel. Canonical images are not produced here (the whole-warp kernel serves those calls).
// ---------------------------------------------------------------------------------------
#ifndef XS_HQ_LPS
#define XS_HQ_LPS 8           // lanes per segment (tools/variants.py)
#endif
constexpr int HQ_LPS = XS_HQ_LPS, HQ_SEGS = 32 / HQ_LPS;

template <class F>
__device__ __noinline__ uint32_t h16q_classify(const uint16_t* xs, uint64_t len, int hl) {
    uint32_t f = 0;
    for (uint64_t i = hl; i < len; i += HQ_LPS) f |= h16_special_flags<F>(__ldg(xs + i));
    return f;
}

template <class F>
__global__ void __launch_bounds__(SSEG_WARPS * 32, XS_SSEG_MINB)
k_segments_h16q(const uint16_t* __restrict__ x, uint64_t nseg, uint64_t seg_len, SegOut o, uint32_t one,
                uint32_t mone) {
    using S = H16Col<F>;
    extern __shared__ __align__(16) int64_t win[];
    __shared__ int64_t gsum[SSEG_WARPS][HQ_SEGS][S::COLS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, hl = lane & (HQ_LPS - 1), grp = lane / HQ_LPS;
    int64_t* col = win + warp * (S::COLS * 32) + lane;
    const int64_t* wb = win + warp * (S::COLS * 32);
    uint32_t* bins = reinterpret_cast<uint32_t*>(win + SSEG_WARPS * S::COLS * 32) + warp * (F::NBIN * 32) + lane;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(bins);
    const uint32_t sbase2 = sbase * 0x00010001u;
    constexpr int SU = SSEG_U;
    constexpr uint32_t WIN_STEPS = F::FLUSH / (SU * 8);           // steps of SU vectors (8 elements each) per bin window
    static_assert(WIN_STEPS >= 1, "window shorter than one step");
#pragma unroll
    for (int j = 0; j < S::COLS; ++j) col[j * 32] = 0;
#pragma unroll
    for (int j = 0; j < F::NBIN; ++j) bins[j * 32] = 0;
    const uint64_t nvec = seg_len / 8;
    const uint64_t nquads = (nseg + HQ_SEGS - 1) / HQ_SEGS;
    const uint64_t nw = (uint64_t)gridDim.x * SSEG_WARPS;
    for (uint64_t qd = (uint64_t)blockIdx.x * SSEG_WARPS + warp; qd < nquads; qd += nw) {
        const uint64_t s = qd * HQ_SEGS + grp;
        const bool mine = s < nseg;
        const uint64_t nv = mine ? nvec : 0;
        const uint4* body = reinterpret_cast<const uint4*>(x + (mine ? s : 0) * seg_len);
        uint32_t steps = 0, flushes = 0, nflush = 0;
        bool special = false;
        uint4 cur[SU], nxt[SU];
        auto load = [&](uint4 (&b)[SU], uint64_t v0) {
            const uint4* p = body + v0 + hl;
            if (v0 + (uint64_t)SU * HQ_LPS <= nv) {                // a whole step: no per-vector guards
#pragma unroll
                for (int u = 0; u < SU; ++u) b[u] = ldg_stream(p + u * HQ_LPS);
            } else {
#pragma unroll
                for (int u = 0; u < SU; ++u)
                    b[u] = v0 + (uint64_t)u * HQ_LPS + hl < nv ? ldg_stream(p + u * HQ_LPS) : make_uint4(0, 0, 0, 0);
            }
        };
        // zero words decode to +0 (bin of group 0, value 0): padding vectors add nothing
        constexpr uint64_t STEP = (uint64_t)SU * HQ_LPS;
        if (nv) load(cur, 0);
        for (uint64_t v0 = 0; v0 < nv; v0 += STEP) {
            if (v0 + STEP < nv) load(nxt, v0 + STEP);
#pragma unroll
            for (int u = 0; u < SU; ++u) {
                h16_add_word<F>(sbase, sbase2, cur[u].x, one, mone);
                h16_add_word<F>(sbase, sbase2, cur[u].y, one, mone);
                h16_add_word<F>(sbase, sbase2, cur[u].z, one, mone);
                h16_add_word<F>(sbase, sbase2, cur[u].w, one, mone);
            }
            if (++steps == WIN_STEPS) {
                special |= h16_flush_col<F>(bins, col);
                steps = 0;
                ++nflush;
                if (++flushes == S::REG_FLUSHES) { h16_col_regularize<F>(col); flushes = 0; }
            }
#pragma unroll
            for (int u = 0; u < SU; ++u) cur[u] = nxt[u];
        }
        special |= h16_flush_col<F>(bins, col);
        // more than one flush: regularize so that the sum of 8 columns stays far inside int64
        if (__any_sync(FULL, nflush > 0)) h16_col_regularize<F>(col);
        uint32_t flags = 0;
        const uint32_t sp = __ballot_sync(FULL, special);
        if (sp) {                                                  // rare: classify NaN / +-Inf (R10)
            if ((sp >> (grp * HQ_LPS)) & ((1u << HQ_LPS) - 1u)) flags = h16q_classify<F>(x + s * seg_len, seg_len, hl);
#pragma unroll
            for (int d = 1; d < HQ_LPS; d <<= 1) flags |= __shfl_xor_sync(FULL, flags, d);   // within the group
        }
        __syncwarp();
        // the group's 8 columns, row by row (raw digits; rows are digits COL0 + r)
        for (int r = hl; r < S::COLS; r += HQ_LPS) {
            int64_t acc = 0;
#pragma unroll
            for (int c = 0; c < HQ_LPS; ++c) acc += wb[r * 32 + grp * HQ_LPS + ((c + hl) & (HQ_LPS - 1))];
            gsum[warp][grp][r] = acc;
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < S::COLS; ++j) col[j * 32] = 0;
        if (hl == 0 && mine) {
            LaneTop t = lane_top_chain<1>(gsum[warp][grp], 0, S::COLS - 1);
            if (t.m >= 0) t.m += S::COL0;
            lane_store_top(t, nullptr, flags, o, s);
        }
        __syncwarp();
    }
}

// Equal binary32 segments (16-B aligned, length a multiple of 4), a quarter warp per segment: the
// same structure as k_segments_h16q with K9's 64-bit exponent-group bins (one read-modify-write per
// element, emptied every SSEG_FLUSH adds). NaN/Inf patterns are summed as finite and a group that
// saw one rescans its segment, cancelling them in its lanes' bins.
template <class F>
__device__ __noinline__ void smallq_rescan(uint64_t* bins, int64_t* col, const uint4* body, uint64_t nvec, int hl,
                                           uint32_t& flags, uint32_t one) {
    uint32_t dummy = 0, adds = 0, flushes = 0;
    scol_regularize<F>(col);                            // fresh headroom for the flushes below
    for (uint64_t v = hl; v < nvec; v += HQ_LPS) {
        const uint4 q = ldg_stream(body + v);
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t f = sspecial_flags<F>(w[i]);
            if (f) {
                flags |= f;
                sbin_add<F>(bins, w[i] ^ (1u << (F::t + F::l)), dummy, one);
                if (++adds == SSEG_FLUSH) {
                    sbin_flush<F>(bins, col);
                    adds = 0;
                    if (++flushes == SSEG_REG_FLUSHES) { scol_regularize<F>(col); flushes = 0; }
                }
            }
        }
    }
    sbin_flush<F>(bins, col);
}

template <class F>
__global__ void __launch_bounds__(SSEG_WARPS * 32, XS_SSEG_MINB)
k_segments_smallq(const float* __restrict__ x, uint64_t nseg, uint64_t seg_len, SegOut o, uint32_t one) {
    extern __shared__ __align__(16) int64_t win[];
    __shared__ int64_t gsum[SSEG_WARPS][HQ_SEGS][F::COLS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, hl = lane & (HQ_LPS - 1), grp = lane / HQ_LPS;
    int64_t* col = win + warp * (F::COLS * 32) + lane;
    const int64_t* wb = win + warp * (F::COLS * 32);
    uint64_t* bins = reinterpret_cast<uint64_t*>(win + SSEG_WARPS * F::COLS * 32) + warp * (F::NBIN * 32) + lane;
    constexpr int SU = SSEG_U;
    constexpr uint32_t WIN_STEPS = SSEG_FLUSH / (SU * 4);        // steps of SU vectors (4 elements each)
#pragma unroll
    for (int j = 0; j < F::COLS; ++j) col[j * 32] = 0;
#pragma unroll
    for (int j = 0; j < F::NBIN; ++j) bins[j * 32] = 0;
    const uint64_t nvec = seg_len / 4;
    const uint64_t nquads = (nseg + HQ_SEGS - 1) / HQ_SEGS;
    const uint64_t nw = (uint64_t)gridDim.x * SSEG_WARPS;
    for (uint64_t qd = (uint64_t)blockIdx.x * SSEG_WARPS + warp; qd < nquads; qd += nw) {
        const uint64_t s = qd * HQ_SEGS + grp;
        const bool mine = s < nseg;
        const uint64_t nv = mine ? nvec : 0;
        const uint4* body = reinterpret_cast<const uint4*>(x + (mine ? s : 0) * seg_len);
        uint32_t steps = 0, flushes = 0, nflush = 0, spec = 0;
        uint4 cur[SU], nxt[SU];
        auto load = [&](uint4 (&b)[SU], uint64_t v0) {
            const uint4* p = body + v0 + hl;
            if (v0 + (uint64_t)SU * HQ_LPS <= nv) {
#pragma unroll
                for (int u = 0; u < SU; ++u) b[u] = ldg_stream(p + u * HQ_LPS);
            } else {
#pragma unroll
                for (int u = 0; u < SU; ++u)
                    b[u] = v0 + (uint64_t)u * HQ_LPS + hl < nv ? ldg_stream(p + u * HQ_LPS) : make_uint4(0, 0, 0, 0);
            }
        };
        constexpr uint64_t STEP = (uint64_t)SU * HQ_LPS;
        if (nv) load(cur, 0);
        for (uint64_t v0 = 0; v0 < nv; v0 += STEP) {
            if (v0 + STEP < nv) load(nxt, v0 + STEP);
#pragma unroll
            for (int u = 0; u < SU; ++u) sbin_add_vec<F>(bins, cur[u], spec, one);   // +0 patterns add 0
            if (++steps == WIN_STEPS) {
                sbin_flush<F>(bins, col);
                steps = 0;
                ++nflush;
                if (++flushes == SSEG_REG_FLUSHES) { scol_regularize<F>(col); flushes = 0; }
            }
#pragma unroll
            for (int u = 0; u < SU; ++u) cur[u] = nxt[u];
        }
        sbin_flush<F>(bins, col);
        uint32_t flags = 0;
        const uint32_t sp = __ballot_sync(FULL, spec == F::EM);
        if (sp) {                                                  // rare: NaN/Inf patterns (R10)
            if ((sp >> (grp * HQ_LPS)) & ((1u << HQ_LPS) - 1u)) {
                smallq_rescan<F>(bins, col, body, nv, hl, flags, one);
                ++nflush;
            }
#pragma unroll
            for (int d = 1; d < HQ_LPS; d <<= 1) flags |= __shfl_xor_sync(FULL, flags, d);   // within the group
        }
        // after more than one flush, regularize: the sum of the group's columns stays far inside int64
        if (__any_sync(FULL, nflush > 0)) scol_regularize<F>(col);
        __syncwarp();
        for (int r = hl; r < F::COLS; r += HQ_LPS) {
            int64_t acc = 0;
#pragma unroll
            for (int c = 0; c < HQ_LPS; ++c) acc += wb[r * 32 + grp * HQ_LPS + ((c + hl) & (HQ_LPS - 1))];
            gsum[warp][grp][r] = acc;
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < F::COLS; ++j) col[j * 32] = 0;
        if (hl == 0 && mine) {
            LaneTop t = lane_top_chain<1>(gsum[warp][grp], 0, F::COLS - 1);
            if (t.m >= 0) t.m += F::COL0;
            lane_store_top(t, nullptr, flags, o, s);
        }
        __syncwarp();
    }
}

template <class F>
static cudaError_t launch_smallq(const void* x, uint64_t nseg, uint64_t seg_len, const SegOut& o, int num_sms,
                                 cudaStream_t s) {
    static unsigned long long smem_set = 0;
    if (cudaError_t e = ensure_smem(k_segments_smallq<F>, sseg_smem<F>(), smem_set)) return e;
    const uint64_t nquads = (nseg + HQ_SEGS - 1) / HQ_SEGS;
    const uint64_t want = (nquads + SSEG_WARPS - 1) / SSEG_WARPS;
    const uint64_t cap = (uint64_t)num_sms * XS_SSEG_MINB;
    const unsigned g = (unsigned)(want < cap ? (want ? want : 1) : cap);
    k_segments_smallq<F><<<g, SSEG_WARPS * 32, sseg_smem<F>(), s>>>(static_cast<const float*>(x), nseg, seg_len, o,
                                                                     1u);
    note_launch();
    return cudaGetLastError();
}

template <class F>
static cudaError_t launch_h16q(const void* x, uint64_t nseg, uint64_t seg_len, const SegOut& o, int num_sms,
                               cudaStream_t s) {
    static unsigned long long smem_set = 0;
    if (cudaError_t e = ensure_smem(k_segments_h16q<F>, h16seg_smem<F>(), smem_set)) return e;
    const uint64_t nquads = (nseg + HQ_SEGS - 1) / HQ_SEGS;
    const uint64_t want = (nquads + SSEG_WARPS - 1) / SSEG_WARPS;
    const uint64_t cap = (uint64_t)num_sms * XS_SSEG_MINB;
    const unsigned g = (unsigned)(want < cap ? (want ? want : 1) : cap);
    k_segments_h16q<F><<<g, SSEG_WARPS * 32, h16seg_smem<F>(), s>>>(static_cast<const uint16_t*>(x), nseg, seg_len, o,
                                                                     1u, 0xFFFFFFFFu);
    note_launch();
    return cudaGetLastError();
}

template <class F>
static cudaError_t launch_h16seg(const void* x, uint64_t nseg, uint64_t seg_len, const uint64_t* offsets,
                                 const SegOut& o, int num_sms, cudaStream_t s, unsigned long long* ticket) {
    static unsigned long long smem_set = 0;
    if (cudaError_t e = ensure_smem(k_segments_h16<F>, h16seg_smem<F>(), smem_set)) return e;
    const uint64_t want = (nseg + SSEG_WARPS - 1) / SSEG_WARPS;
    const uint64_t cap = (uint64_t)num_sms * XS_SSEG_MINB;
    const unsigned g = (unsigned)(want < cap ? (want ? want : 1) : cap);
    k_segments_h16<F><<<g, SSEG_WARPS * 32, h16seg_smem<F>(), s>>>(static_cast<const uint16_t*>(x), nseg, seg_len,
                                                                    offsets, o, offsets ? ticket : nullptr, 1u,
                                                                    0xFFFFFFFFu);
    note_launch();
    return cudaGetLastError();
}

template <class F>
static cudaError_t launch_small(const void* x, uint64_t nseg, uint64_t seg_len, const uint64_t* offsets,
                                const SegOut& o, int num_sms, cudaStream_t s, unsigned long long* ticket) {
    static unsigned long long smem_set = 0;
    if (cudaError_t e = ensure_smem(k_segments_small<F>, sseg_smem<F>(), smem_set)) return e;
    const uint64_t want = (nseg + SSEG_WARPS - 1) / SSEG_WARPS;
    const uint64_t cap = (uint64_t)num_sms * XS_SSEG_MINB;
    const unsigned g = (unsigned)(want < cap ? (want ? want : 1) : cap);
    k_segments_small<F><<<g, SSEG_WARPS * 32, sseg_smem<F>(), s>>>(static_cast<const uint8_t*>(x), nseg, seg_len,
                                                                    offsets, o, offsets ? ticket : nullptr, 1u);
    note_launch();
    return cudaGetLastError();
}

#ifndef XS_H16Q
#define XS_H16Q 1             // quarter-warp 16-bit segments (tools/variants.py: 0 = whole warps)
#endif
static bool h16q_ok(const void* x, uint64_t seg_len, const uint64_t* offsets, const SegOut& o) {
    return XS_H16Q && !offsets && !o.canon && seg_len >= 8 && seg_len % 8 == 0 && ((uintptr_t)x & 15) == 0;
}

cudaError_t sum_segments_small(const void* x, int dtype, uint64_t nseg, uint64_t seg_len, const uint64_t* offsets,
                               const SegOut& o, int num_sms, cudaStream_t s, unsigned long long* ticket) {
    if (!offsets && seg_len > 0 && seg_len <= SEG_LANES_MAX)
        return sum_segments_lanes(x, dtype, nseg, seg_len, o, num_sms, s);
    switch (dtype) {
        case XSUM_DT_F32:
            if (XS_H16Q && !offsets && !o.canon && seg_len >= 4 && seg_len % 4 == 0 && ((uintptr_t)x & 15) == 0)
                return launch_smallq<SF32>(x, nseg, seg_len, o, num_sms, s);
            return launch_small<SF32>(x, nseg, seg_len, offsets, o, num_sms, s, ticket);
        case XSUM_DT_F16:
            if (h16q_ok(x, seg_len, offsets, o)) return launch_h16q<FmtF16>(x, nseg, seg_len, o, num_sms, s);
            return launch_h16seg<FmtF16>(x, nseg, seg_len, offsets, o, num_sms, s, ticket);
        case XSUM_DT_BF16:
            if (h16q_ok(x, seg_len, offsets, o)) return launch_h16q<FmtBF16Q>(x, nseg, seg_len, o, num_sms, s);
            return launch_h16seg<FmtBF16Seg>(x, nseg, seg_len, offsets, o, num_sms, s, ticket);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace xs
