// K6: segmented exact sums (BASELINE.json config 5) and CSR variable-length segments.
//
// One warp reduces one segment with the same lane-column hot loop as K2, then combines
// its 32 columns, regularizes and rounds without
// leaving the warp - the paper's per-partition "combine" with a
// warp as the partition's worker. Warps loop over segments (persistent grid): equal segments
// in a fixed order, CSR segments in the order they draw them from a ticket word (dynamic
// balancing of ragged lengths). Equal segments of <= SEG_LANES_MAX elements go to K11
// (segments_lanes.cu: one lane per segment).
#include <cuda_runtime.h>

#include "band_round.cuh"
#include "xsum_device.cuh"
#include "xsum_kernels.h"

namespace xs {

#ifndef XS_SEGU_WARPS
#define XS_SEGU_WARPS 8   // k_segments_uniform: warps per block, XS_SEGU_MINB blocks per SM
#endif
#ifndef XS_SEGU_MINB
#define XS_SEGU_MINB 2
#endif
constexpr int SEG_WARPS = XS_SEGU_WARPS;
#ifndef XS_SEG_U
#define XS_SEG_U 4
#endif
constexpr int SEG_U = XS_SEG_U;
constexpr int SEG_FLUSH_ITERS = FLUSH_ELEMS / (2 * SEG_U);
constexpr size_t SEG_SMEM = (size_t)SEG_WARPS * D * 32 * sizeof(int64_t);

__device__ __noinline__ void seg_rescan(int64_t* col, const uint4* body, uint64_t it0, uint64_t it1, int lane,
                                           uint32_t& flags, uint32_t one) {
    for (uint64_t it = it0; it <= it1; ++it) {
#pragma unroll
        for (int u = 0; u < SEG_U; ++u) {
            uint4 v = ldg_stream(body + it * (32 * SEG_U) + u * 32 + lane);
            column_fix_special(col, v.x, v.y, flags, one);
            column_fix_special(col, v.z, v.w, flags, one);
        }
    }
}

// Per-segment epilogue of K6's CSR loop (one warp): combine the 32 lane columns (|sum| <= 32 (2^51 +
// 2^11) < 2^57), regularize, canonicalize and round and write
// the outputs, reading (and zeroing behind itself) only the rows the segment can
// have touched: every chunk of a summand with exponent index k lands in digits <= k / 52 + 1, and
// a column that was regularized inside the segment (long segments only) may hold carries up to
// digit D-1, so rows 32..41 are read when top = max over the warp of those bounds reaches 32
// (c5csr's exponents reach digit 25: one row per lane). The rest of the column is zero.
__device__ __forceinline__ void segment_epilogue_top(int64_t* wb, int64_t* su, uint32_t flags, int top,
                                                     uint64_t len, uint64_t s, const SegOut& o, int lane) {
    __syncwarp();
    if (!o.canon && top < 31) {
        // values only, every chunk in rows <= top < 31 (the top carry lands in row top + 1 <= 31):
        // one row per lane, read straight-line (column lane ^ c at step c: a conflict-free
        // permutation) and zeroed, then the per-slot regularization / canonicalization / rounding
        // of band_round.cuh with the whole warp as one slot of 32 digits (LPS = 32, NK = 1).
        SlotSums<32> d;
        d.hs[0] = d.ls[0] = d.hs[1] = d.ls[1] = 0;
        if (lane <= top) {
            int64_t* row = wb + lane * 32;
#pragma unroll
            for (int c0 = 0; c0 < 32; c0 += 8) {
                int64_t v[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) v[c] = row[lane ^ (c0 + c)];
#pragma unroll
                for (int c = 0; c < 8; ++c) row[lane ^ (c0 + c)] = 0;
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    d.hs[0] += v[c] >> 32;
                    d.ls[0] += (int64_t)(uint32_t)v[c];
                }
            }
        }
        __syncwarp();
        int64_t a[SlotSums<32>::KD];
        slot_digits<32, 1>(d, a, lane, 0);
        flags = __reduce_or_sync(FULL, flags);
        xsum_result r = slot_finalize<32, 1>(a, flags, len, nullptr, su, lane, 0, 0);
        if (lane == 0) o.write(s, r);
        return;
    }
    LaneSums t = {0, 0, 0, 0};
    const bool hi_rows = top >= 32;                  // warp-uniform
#pragma unroll 8
    for (int c = 0; c < 32; ++c) {
        const int cc = (lane + c) & 31;              // rotated: conflict-free columns
        const int64_t v0 = wb[lane * 32 + cc];
        wb[lane * 32 + cc] = 0;
        t.hs0 += v0 >> 32;
        t.ls0 += (int64_t)(uint32_t)v0;
        if (hi_rows && lane + 32 < D) {
            const int64_t v1 = wb[(lane + 32) * 32 + cc];
            wb[(lane + 32) * 32 + cc] = 0;
            t.hs1 += v1 >> 32;
            t.ls1 += (int64_t)(uint32_t)v1;
        }
    }
    __syncwarp();
    int64_t a0, a1;
    sums_to_digits(t, a0, a1, lane);
    flags = __reduce_or_sync(FULL, flags);
    // inline (finalize_warp_inl): an out-of-line call would wait for the next segment's loads
    xsum_result r = finalize_warp_inl(a0, a1, flags, len, o.canon ? o.canon + s * XSUM_CANON_LIMBS : nullptr, su, lane);
    if (lane == 0) o.write(s, r);
}

// exponent index k = max(e, 1) - 1 of a binary64 high word (its chunks land in digits <= k / 52 + 1)
__device__ __forceinline__ uint32_t kidx(uint32_t hi) { return max((hi >> 20) & 0x7FFu, 1u) - 1u; }

#ifndef XS_SEGC_WARPS
#define XS_SEGC_WARPS 16  // one 16-warp block per SM (c5csr 549 vs 544 G/s for two 8-warp blocks)
#endif
#ifndef XS_SEGC_MINB
#define XS_SEGC_MINB 1
#endif
#ifndef XS_SEGC_NB
#define XS_SEGC_NB 2      // rotating tile buffers of the CSR loop
#endif
constexpr int SEGC_WARPS = XS_SEGC_WARPS;
constexpr int SEGC_NB = XS_SEGC_NB;
constexpr size_t SEGC_SMEM = (size_t)SEGC_WARPS * D * 32 * sizeof(int64_t);

__global__ void __launch_bounds__(SEGC_WARPS * 32, XS_SEGC_MINB)
k_segments(const double* __restrict__ x, uint64_t nseg, uint64_t seg_len, const uint64_t* __restrict__ offsets,
           SegOut o, unsigned long long* __restrict__ ticket, uint32_t one, uint32_t mone) {
    extern __shared__ __align__(16) int64_t win[];
    __shared__ int64_t su[SEGC_WARPS][64];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t* col = win + warp * (D * 32) + lane;
    const uint64_t nw = (uint64_t)gridDim.x * SEGC_WARPS;

    // A warp's segments s, s + nw, ...: the next segment's bounds and first tile are fetched
    // before the current segment's epilogue, so its DRAM latency hides behind the epilogue.
    struct Seg {
        const double* xs;
        uint64_t len, head, nbody, nvec, nit;
        const uint4* body;
    };
    // CSR bounds of the segment after next are loaded one segment ahead (ob, oe)
    auto bounds = [&](uint64_t sj, uint64_t& b, uint64_t& e) {
        if (sj < nseg) {
            b = offsets ? __ldg(offsets + sj) : sj * seg_len;
            e = offsets ? __ldg(offsets + sj + 1) : b + seg_len;
        }
    };
    auto open_seg = [&](uint64_t beg, uint64_t end) {
        Seg g;
        g.len = end - beg;
        g.xs = x + beg;
        g.head = (g.len && ((uintptr_t)g.xs & 15)) ? 1 : 0;
        g.nbody = g.len - g.head;
        g.nvec = g.nbody >> 1;
        g.body = reinterpret_cast<const uint4*>(g.xs + g.head);
        g.nit = g.nvec / (32 * SEG_U);
        return g;
    };
    // Segment order: with a ticket counter, warps take the next unclaimed segment (dynamic
    // balancing: ragged CSR lengths made the static round-robin's busiest warp do 1.36x the mean
    // work on c5csr); without one, segments s, s + nw, ... (static).
    uint64_t s = ticket ? seg_next(ticket, 0, nw, lane) : (uint64_t)blockIdx.x * SEGC_WARPS + warp;
    if (s >= nseg) return;                                           // warp-uniform
#pragma unroll
    for (int j = 0; j < D; ++j) col[j * 32] = 0;
    uint64_t cb = 0, ce = 0, ob = 0, oe = 0;
    bounds(s, cb, ce);
    Seg g = open_seg(cb, ce);
    // SEGC_NB register buffers rotate without moves (tile t of a segment in buf[t % SEGC_NB]): while
    // one tile is decoded the next SEGC_NB - 1 are in flight; the first SEGC_NB - 1 tiles of the next
    // segment are fetched before the current segment's epilogue
    uint4 buf[SEGC_NB][SEG_U];
    auto load_tile = [&](uint4 (&bf)[SEG_U], const uint4* body, uint64_t t) {
#pragma unroll
        for (int u = 0; u < SEG_U; ++u) bf[u] = ldg_stream(body + t * (32 * SEG_U) + u * 32 + lane);
    };
#pragma unroll
    for (int b = 0; b < SEGC_NB - 1; ++b)
        if ((uint64_t)b < g.nit) load_tile(buf[b], g.body, b);
    while (true) {
        const uint64_t sn = seg_next(ticket, s, nw, lane);
        bounds(sn, ob, oe);                                          // next segment's bounds, early
        uint32_t flags = 0, nspec = 0, kmax = 0;
        bool flushed = false;
        const uint64_t nit = g.nit, nvec = g.nvec;
        const uint4* body = g.body;
        uint64_t wstart = 0;
        int since = 0;
        auto process = [&](const uint4 (&bf)[SEG_U], uint64_t it) {
#pragma unroll
            for (int u = 0; u < SEG_U; ++u) {
                Chunks a = decompose(bf[u].x, bf[u].y, one, mone);
                nspec = spec_fold(nspec, a);
                column_add(col, a, one);
                Chunks b = decompose(bf[u].z, bf[u].w, one, mone);
                nspec = spec_fold(nspec, b);
                column_add(col, b, one);
            }
            if (++since == SEG_FLUSH_ITERS) {
                regularize_column(col);
                flushed = true;
                if (__any_sync(FULL, spec_hit(nspec))) {
                    if (spec_hit(nspec)) {
                        seg_rescan(col, body, wstart, it, lane, flags, one);
                        regularize_column(col);
                    }
                }
                kmax = max(kmax, nspec);
                nspec = 0;
                since = 0;
                wstart = it + 1;
            }
        };
        for (uint64_t it = 0; it < nit; it += SEGC_NB) {
#pragma unroll
            for (int b = 0; b < SEGC_NB; ++b) {
                if (it + b >= nit) break;                            // warp-uniform
                if (it + b + SEGC_NB - 1 < nit) load_tile(buf[(b + SEGC_NB - 1) % SEGC_NB], body, it + b + SEGC_NB - 1);
                process(buf[b], it + b);
            }
        }
        // leftover vectors (issued together before use), head and tail: checked adds
        uint4 lv[SEG_U];
#pragma unroll
        for (int u = 0; u < SEG_U; ++u) {
            const uint64_t v = nit * (32 * SEG_U) + u * 32 + lane;
            if (v < nvec) lv[u] = ldg_stream(body + v);
        }
#pragma unroll
        for (int u = 0; u < SEG_U; ++u) {
            if (nit * (32 * SEG_U) + u * 32 + lane < nvec) {
                column_add_checked(col, lv[u].x, lv[u].y, flags, one);
                column_add_checked(col, lv[u].z, lv[u].w, flags, one);
                kmax = max(kmax, max(kidx(lv[u].y), kidx(lv[u].w)));
            }
        }
        if (lane == 0 && g.head) {
            uint2 q = ldg_one(g.xs);
            column_add_checked(col, q.x, q.y, flags, one);
            kmax = max(kmax, kidx(q.y));
        }
        if (lane == 1 && (g.nbody & 1)) {
            uint2 q = ldg_one(g.xs + g.head + 2 * nvec);
            column_add_checked(col, q.x, q.y, flags, one);
            kmax = max(kmax, kidx(q.y));
        }
        if (__any_sync(FULL, spec_hit(nspec))) {        // raw columns go to the epilogue
            if (spec_hit(nspec) && since) {
                regularize_column(col);
                seg_rescan(col, body, wstart, nit - 1, lane, flags, one);
            }
        }
        // prefetch the next segment, then close this one (the epilogue zeroes the columns)
        const bool more = sn < nseg;
        const uint64_t len = g.len;
        if (more) {
            g = open_seg(ob, oe);
#pragma unroll
            for (int b = 0; b < SEGC_NB - 1; ++b)
                if ((uint64_t)b < g.nit) load_tile(buf[b], g.body, b);
        }
        // checked adds of the head / tail / leftovers may reach any digit: include them
        int top = flushed ? D : (int)(max(kmax, nspec) / 52u) + 1;
        top = __reduce_max_sync(FULL, top);
        segment_epilogue_top(win + warp * (D * 32), su[warp], flags, top, len, s, o, lane);
        if (!more) break;
        s = sn;
    }
}


// Fast path for equal segments whose starts are 16-B aligned and whose length is a multiple
// of one warp tile (256 doubles), e.g. config 5: a warp's tiles form one continuous stream
// across its segments, loaded SEG_NB - 1 tiles ahead into rotating register buffers, so the
// per-segment epilogue runs while the next segment's first loads are already in flight.
// (profiles/r01_c5_diagnosis.txt: deeper buffers, dedicated epilogue warps and 128-bit
// column-sum loads were measured and are not faster.)
constexpr uint32_t SEG_TILE = 32 * SEG_U * 2;   // doubles per warp tile
#ifndef XS_SEG_NB
#define XS_SEG_NB 2   // streaming path needs tiles-per-segment % NB == 0; c5: NB=2 597, NB=4 585 G/s
#endif
constexpr int SEG_NB = XS_SEG_NB;               // rotating register buffers (SEG_NB-1 tiles in flight)

__device__ __noinline__ void seg_rescan_uniform(int64_t* col, const uint4* seg, uint32_t t0, uint32_t t1,
                                                   int lane, uint32_t& flags, uint32_t one) {
    for (uint32_t t = t0; t <= t1; ++t) {
#pragma unroll
        for (int u = 0; u < SEG_U; ++u) {
            uint4 v = ldg_stream(seg + (uint64_t)t * (32 * SEG_U) + u * 32 + lane);
            column_fix_special(col, v.x, v.y, flags, one);
            column_fix_special(col, v.z, v.w, flags, one);
        }
    }
}

__global__ void __launch_bounds__(SEG_WARPS * 32, XS_SEGU_MINB)
k_segments_uniform(const double* __restrict__ x, uint64_t nseg, uint64_t seg_len, SegOut o, uint32_t one,
                   uint32_t mone) {
    extern __shared__ __align__(16) int64_t win[];
    __shared__ int64_t su[SEG_WARPS][64];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t* col = win + warp * (D * 32) + lane;
    const uint64_t nw = (uint64_t)gridDim.x * SEG_WARPS;
    const uint64_t gw = (uint64_t)blockIdx.x * SEG_WARPS + warp;
    if (gw >= nseg) return;                                    // warp-uniform
    const uint32_t TPS = (uint32_t)(seg_len / SEG_TILE);       // tiles per segment
    const uint64_t seg_vecs = seg_len / 2;
    const uint4* xv = reinterpret_cast<const uint4*>(x);
#pragma unroll
    for (int j = 0; j < D; ++j) col[j * 32] = 0;

    // Load cursor: TPS is a multiple of SEG_NB (dispatch condition), so an NB-tile group never
    // crosses a segment: one bounds check and one segment step per group, pointer increments
    // only (no 64-bit multiplies on the hot path).
    constexpr uint32_t TV = 32 * SEG_U;                        // vectors per warp tile
    const uint64_t seg_skip = (nw - 1) * seg_vecs;             // from a segment's end to this warp's next
    const uint4* lp = xv + gw * seg_vecs + lane;
    uint64_t ls = gw;
    uint32_t lt = 0;
    auto advance_load = [&]() {
        lp += SEG_NB * TV;
        lt += SEG_NB;
        if (lt == TPS) { lt = 0; ls += nw; lp += seg_skip; }
    };
    uint64_t ps = gw;            // processing cursor: segment, tile
    uint32_t pt = 0, wstart = 0, flags = 0, nspec = 0;
    int groups = 0;
    // The lane columns are never zeroed: a segment's digits are the difference of the raw lane
    // sums at its end and at the previous segment's end (exact integer arithmetic; the
    // regularizations in between preserve every column's value, so the digit-wise difference
    // still represents exactly the value this segment added).
    LaneSums prev = {0, 0, 0, 0};
    constexpr int GROUPS_PER_WINDOW = SEG_FLUSH_ITERS / SEG_NB;
    uint4 buf[SEG_NB][SEG_U];
#pragma unroll
    for (int b = 0; b < SEG_NB; ++b)
#pragma unroll
        for (int u = 0; u < SEG_U; ++u) buf[b][u] = ldg_stream(lp + b * TV + u * 32);
    advance_load();
    while (ps < nseg) {
        const bool ld = ls < nseg;
#pragma unroll
        for (int b = 0; b < SEG_NB; ++b) {
#pragma unroll
            for (int u = 0; u < SEG_U; ++u) {
#ifdef XS_EXP_SEG_NOACC   // diagnostic (wrong sums): loads only
                nspec ^= buf[b][u].x ^ buf[b][u].y ^ buf[b][u].z ^ buf[b][u].w;
#else
                Chunks a = decompose(buf[b][u].x, buf[b][u].y, one, mone);
                nspec = spec_fold(nspec, a);
                column_add(col, a, one);
                Chunks c = decompose(buf[b][u].z, buf[b][u].w, one, mone);
                nspec = spec_fold(nspec, c);
                column_add(col, c, one);
#endif
            }
            if (ld) {
#pragma unroll
                for (int u = 0; u < SEG_U; ++u) buf[b][u] = ldg_stream(lp + b * TV + u * 32);
            }
        }
        if (ld) advance_load();
        pt += SEG_NB;
        ++groups;
        if (pt == TPS) {                                       // segment complete
            if (__any_sync(FULL, spec_hit(nspec))) {           // rare: cancel NaN/Inf patterns
                if (spec_hit(nspec)) {
                    regularize_column(col);
                    seg_rescan_uniform(col, xv + ps * seg_vecs, wstart, pt - 1, lane, flags, one);
                    regularize_column(col);
                }
                nspec = 0;
                groups = 0;                                    // the window restarts (all lanes)
            }
            // epilogue inline: an out-of-line call would wait for the in-flight buffers
#if defined(XS_EXP_SEG_NOEPI) || defined(XS_EXP_SEG_NOACC)   // diagnostic (wrong sums)
            if (lane == 0) o.out[ps] = (double)nspec;
            if (false) {
#else
            {
#endif
            const int64_t* wb = win + warp * (D * 32);
            __syncwarp();
            LaneSums now = raw_lane_sums(wb, lane);
            LaneSums d = {now.hs0 - prev.hs0, now.ls0 - prev.ls0, now.hs1 - prev.hs1, now.ls1 - prev.ls1};
            prev = now;
            int64_t a0, a1;
            sums_to_digits(d, a0, a1, lane);
            const uint32_t fl = __reduce_or_sync(FULL, flags);
            xsum_result r = finalize_warp_inl(a0, a1, fl, seg_len, o.canon ? o.canon + ps * XSUM_CANON_LIMBS : nullptr,
                                              su[warp], lane);
            if (lane == 0) o.write(ps, r);
            }
            flags = 0;
            wstart = 0;                                        // window tiles of the next segment start at 0
            pt = 0;
            ps += nw;
        }
        if (groups == GROUPS_PER_WINDOW) {                     // window close (may span segments)
            regularize_column_inl(col);
            if (__any_sync(FULL, spec_hit(nspec))) {           // pending only in the current segment
                if (spec_hit(nspec)) {
                    seg_rescan_uniform(col, xv + ps * seg_vecs, wstart, pt - 1, lane, flags, one);
                    regularize_column(col);
                }
            }
            nspec = 0;
            groups = 0;
            wstart = pt;
        }
    }
}

cudaError_t sum_segments(const double* x, uint64_t nseg, uint64_t seg_len, const uint64_t* offsets, const SegOut& o,
                         int num_sms, cudaStream_t s, unsigned long long* ticket) {
    if (!offsets && seg_len > 0 && seg_len <= SEG_LANES_MAX)
        return sum_segments_lanes(x, XSUM_DT_F64, nseg, seg_len, o, num_sms, s);
    static unsigned long long smem_set = 0, smem_set_u = 0;
    if (cudaError_t e = ensure_smem(k_segments, SEGC_SMEM, smem_set)) return e;
    if (cudaError_t e = ensure_smem(k_segments_uniform, SEG_SMEM, smem_set_u)) return e;
    uint64_t want = (nseg + SEG_WARPS - 1) / SEG_WARPS;
    uint64_t cap = (uint64_t)num_sms * XS_SEGU_MINB;
    unsigned g = (unsigned)(want < cap ? (want ? want : 1) : cap);
    const bool uniform = !offsets && seg_len >= SEG_TILE && seg_len % ((uint64_t)SEG_TILE * SEG_NB) == 0 &&
                         ((uintptr_t)x & 15) == 0 && seg_len / SEG_TILE < (1u << 31);
#ifndef XS_SEG_HALF
#define XS_SEG_HALF 1
#endif
    if (XS_SEG_HALF && !offsets && segments_half_ok(x, seg_len))
        return sum_segments_half(x, nseg, seg_len, o, num_sms, s);
    if (uniform)
        k_segments_uniform<<<g, SEG_WARPS * 32, SEG_SMEM, s>>>(x, nseg, seg_len, o, 1u, 0xFFFFFFFFu);
    else {
        const uint64_t wantc = (nseg + SEGC_WARPS - 1) / SEGC_WARPS, capc = (uint64_t)num_sms * XS_SEGC_MINB;
        const unsigned gc = (unsigned)(wantc < capc ? (wantc ? wantc : 1) : capc);
        k_segments<<<gc, SEGC_WARPS * 32, SEGC_SMEM, s>>>(x, nseg, seg_len, offsets, o, offsets ? ticket : nullptr, 1u,
                                                          0xFFFFFFFFu);
    }
    note_launch();
    return cudaGetLastError();
}

}  // namespace xs
