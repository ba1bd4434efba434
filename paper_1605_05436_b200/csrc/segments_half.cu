// K6h: equal binary64 segments with HALF a warp per segment (config 5's streaming path, two
// segments per warp). profiles/r01_c5_diagnosis.txt: the per-segment epilogue (the column
// combine, carry resolution and rounding) costs ~15% of c5 and the loop is
// issue-bound. With 16 lanes per segment the combine reads 16 instead of 32 lane columns per
// segment and the two halves run their epilogues together (16-wide shuffles, ballots split by
// half): the epilogue instructions per segment halve, the streaming loop is K6's (each half
// reads its own segment's rows). The code is generic in the lanes per segment (LPS = 16 kept;
// 8, quarter warps, measured slower: its 6-digit-per-lane epilogue spills).
#include <cuda_runtime.h>

#include "band_round.cuh"
#include "xsum_device.cuh"
#include "xsum_kernels.h"

namespace xs {

#ifndef XS_SH_MINB
#define XS_SH_MINB 1
#endif
#ifndef XS_SH_WARPS
#define XS_SH_WARPS 16     // K6h (segments of > 1008 summands per lane): one 16-warp block per SM (65536-long: 586 -> 606 G/s)
#endif
constexpr int SH_WARPS = XS_SH_WARPS;
#ifndef XS_SH_U
#define XS_SH_U 8
#endif
#ifndef XS_SH_NB
#define XS_SH_NB 2
#endif
#ifndef XS_SH_LPS
#define XS_SH_LPS 16
#endif
constexpr int SH_U = XS_SH_U;                  // 16-B vectors per lane per tile
constexpr int SH_NB = XS_SH_NB;                // rotating tile buffers
constexpr int LPS = XS_SH_LPS;                 // lanes per segment (16: half warps; 8: quarters)
constexpr int SEGS = 32 / LPS;                 // segments per warp at a time
constexpr int KD = (D + LPS - 1) / LPS;        // digits per lane: lane sl holds sl + LPS k
constexpr uint32_t SH_TILE = LPS * SH_U * 2;   // doubles per segment tile
constexpr int SH_FLUSH_TILES = FLUSH_ELEMS / (2 * SH_U);
constexpr size_t SH_SMEM = (size_t)SH_WARPS * D * 32 * sizeof(int64_t);

using HalfSums = SlotSums<LPS>;
__device__ __forceinline__ uint32_t half_bits(uint32_t ballot, int half) { return slot_bits<LPS>(ballot, half); }
template <int NK = KD>
__device__ __forceinline__ void half_digits(const HalfSums& d, int64_t (&a)[KD], int hl, int base = 0) {
    slot_digits<LPS, NK>(d, a, hl, base);
}
template <int NK = KD>
__device__ __forceinline__ xsum_result finalize_half(int64_t (&a)[KD], uint32_t flags, uint64_t count, uint64_t* canon,
                                                     int64_t* su, int hl, int half, int base = 0) {
    return slot_finalize<LPS, NK>(a, flags, count, canon, su, hl, half, base);
}

// Raw lane sums of one half's 16 columns: lane hl sums rows hl, hl+16, hl+32 (hi / lo words
// apart, as raw_lane_sums: |raw| < 2^63).
__device__ __forceinline__ HalfSums half_raw_sums(const int64_t* wb, int hl, int half) {
    HalfSums t;
#pragma unroll
    for (int k = 0; k < KD; ++k) t.hs[k] = t.ls[k] = 0;
#pragma unroll 4
    for (int c = 0; c < LPS; ++c) {
        const int cc = half * LPS + ((hl + c) & (LPS - 1));   // rotated: conflict-free within the slot
#pragma unroll
        for (int k = 0; k < KD; ++k) {
            const int row = hl + LPS * k;
            if (row < D) {
                const int64_t v = wb[row * 32 + cc];
                t.hs[k] += v >> 32;
                t.ls[k] += (int64_t)(uint32_t)v;
            }
        }
    }
    return t;
}

__device__ __noinline__ void half_rescan(int64_t* col, const uint4* seg, uint32_t t0, uint32_t t1, int hl,
                                         uint32_t& flags, uint32_t one) {
    for (uint32_t t = t0; t <= t1; ++t) {
#pragma unroll
        for (int u = 0; u < SH_U; ++u) {
            uint4 v = ldg_stream(seg + (uint64_t)t * (LPS * SH_U) + u * LPS + hl);
            column_fix_special(col, v.x, v.y, flags, one);
            column_fix_special(col, v.z, v.w, flags, one);
        }
    }
}

__global__ void __launch_bounds__(SH_WARPS * 32, XS_SH_MINB)
k_segments_half(const double* __restrict__ x, uint64_t nseg, uint64_t seg_len, SegOut o, uint32_t one, uint32_t mone) {
    extern __shared__ __align__(16) int64_t win[];
    __shared__ int64_t su[SH_WARPS][SEGS][48];
    __shared__ uint64_t canon_sink[SH_WARPS][XSUM_CANON_LIMBS];   // the odd last pair's idle half
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, hl = lane & (LPS - 1), half = lane / LPS;
    int64_t* col = win + warp * (D * 32) + lane;
    const uint64_t nw = (uint64_t)gridDim.x * SH_WARPS;
    const uint64_t npairs = (nseg + SEGS - 1) / SEGS;          // groups of SEGS segments
    const uint64_t gw = (uint64_t)blockIdx.x * SH_WARPS + warp;
    if (gw >= npairs) return;                                  // warp-uniform
    const uint32_t TPS = (uint32_t)(seg_len / SH_TILE);        // half tiles per segment
    const uint64_t seg_vecs = seg_len / 2;
    const uint4* xv = reinterpret_cast<const uint4*>(x);
#pragma unroll
    for (int j = 0; j < D; ++j) col[j * 32] = 0;
    // this half's segments: 2p + half for the warp's pairs p = gw, gw + nw, ...; the second half
    // of a last, odd pair re-reads its partner's segment and writes nothing
    auto seg_of = [&](uint64_t p) -> uint64_t {
        const uint64_t s = SEGS * p + half;
        return s < nseg ? s : SEGS * p;
    };
    constexpr uint32_t TV = LPS * SH_U;
    const uint4* lp = xv + seg_of(gw) * seg_vecs + hl;
    uint64_t lpair = gw;
    uint32_t lt = 0;
    auto advance_load = [&]() {
        lp += SH_NB * TV;
        lt += SH_NB;
        if (lt == TPS) {
            lt = 0;
            lpair += nw;
            lp = xv + seg_of(lpair < npairs ? lpair : gw) * seg_vecs + hl;
        }
    };
    uint64_t pp = gw;
    uint32_t pt = 0, wstart = 0, flags = 0, nspec = 0;
    int groups = 0;
    HalfSums prev;
#pragma unroll
    for (int k = 0; k < KD; ++k) prev.hs[k] = prev.ls[k] = 0;
    constexpr int GROUPS_PER_WINDOW = SH_FLUSH_TILES / SH_NB;
    uint4 buf[SH_NB][SH_U];
#pragma unroll
    for (int bb = 0; bb < SH_NB; ++bb)
#pragma unroll
        for (int u = 0; u < SH_U; ++u) buf[bb][u] = ldg_stream(lp + bb * TV + u * LPS);
    advance_load();
    while (pp < npairs) {
        const bool ld = lpair < npairs;
#pragma unroll
        for (int bb = 0; bb < SH_NB; ++bb) {
#pragma unroll
            for (int u = 0; u < SH_U; ++u) {
                Chunks a = decompose(buf[bb][u].x, buf[bb][u].y, one, mone);
                nspec = spec_fold(nspec, a);
                column_add(col, a, one);
                Chunks c = decompose(buf[bb][u].z, buf[bb][u].w, one, mone);
                nspec = spec_fold(nspec, c);
                column_add(col, c, one);
            }
            if (ld) {
#pragma unroll
                for (int u = 0; u < SH_U; ++u) buf[bb][u] = ldg_stream(lp + bb * TV + u * LPS);
            }
        }
        if (ld) advance_load();
        pt += SH_NB;
        ++groups;
        const uint64_t ps = seg_of(pp);
        if (pt == TPS) {                                       // both halves' segments complete
            if (__any_sync(FULL, spec_hit(nspec))) {
                if (spec_hit(nspec)) {
                    regularize_column(col);
                    half_rescan(col, xv + ps * seg_vecs, wstart, pt - 1, hl, flags, one);
                    regularize_column(col);
                }
                nspec = 0;
                groups = 0;
            }
            const int64_t* wb = win + warp * (D * 32);
            __syncwarp();
            const HalfSums now = half_raw_sums(wb, hl, half);
            HalfSums d;
#pragma unroll
            for (int k = 0; k < KD; ++k) {
                d.hs[k] = now.hs[k] - prev.hs[k];
                d.ls[k] = now.ls[k] - prev.ls[k];
            }
            prev = now;
            int64_t a[KD];
            half_digits(d, a, hl);
            uint32_t fl = flags;
#pragma unroll
            for (int off = LPS / 2; off > 0; off >>= 1) fl |= __shfl_xor_sync(FULL, fl, off, LPS);
            const bool mine = SEGS * pp + half < nseg;
            // canon pointer non-null for both halves or neither (finalize_half syncs the warp in it)
            uint64_t* cp = o.canon ? (mine ? o.canon + ps * XSUM_CANON_LIMBS : canon_sink[warp]) : nullptr;
            xsum_result r = finalize_half(a, fl, seg_len, cp, su[warp][half], hl, half);
            if (hl == 0 && mine) o.write(ps, r);
            flags = 0;
            wstart = 0;
            pt = 0;
            pp += nw;
        }
        if (groups == GROUPS_PER_WINDOW) {
            regularize_column_inl(col);
            if (__any_sync(FULL, spec_hit(nspec))) {
                if (spec_hit(nspec)) {
                    half_rescan(col, xv + seg_of(pp) * seg_vecs, wstart, pt - 1, hl, flags, one);
                    regularize_column(col);
                }
            }
            nspec = 0;
            groups = 0;
            wstart = pt;
        }
    }
}

// ---------------------------------------------------------------------------------
// K6z: the same half-warp streaming loop for segments of at most SZ_MAX_LANE summands per lane
// (c5: 256). Each segment starts from ZEROED lane columns, so no summand count ever needs a
// regularization inside the loop and no raw-sum snapshot of the previous segment is kept (12 fewer
// live registers than K6h: the epilogue reads the columns and zeroes them behind itself). The loop
// tracks the band of exponents the lane saw with ONE packed 16x2 max (lo: max k, hi: 0xFFFF - min k;
// the max also serves as K2's NaN/Inf detector); at the segment's end the half's digit band
// [k_min / 52, k_max / 52 + 1] is the only part of its 16 columns that is combined, zeroed,
// regularized, canonicalized and rounded (positions relative to the band's lowest digit): c5's
// exponents span ~10 of the 42 digits, one row group per lane instead of three.
#ifndef XS_SZ_U
#define XS_SZ_U 8
#endif
#ifndef XS_SZ_NB
#define XS_SZ_NB 2
#endif
// two shapes: U = XS_SZ_U (8) vectors per lane per tile for lengths that are multiples of 2 tiles of
// 256 doubles (c5), U = 4 for the other multiples of 256 (e.g. rows of 768)
constexpr int SZ_U1 = XS_SZ_U, SZ_NB1 = XS_SZ_NB, SZ_U2 = 4;
constexpr uint32_t SZ_GRAN1 = LPS * SZ_U1 * 2 * SZ_NB1, SZ_GRAN2 = LPS * SZ_U2 * 2 * 2;
// per-lane summands per segment: every digit of a zeroed column receives at most one chunk
// (|chunk| <= 2^52) per summand and one per NaN/Inf cancellation: 2 * 1008 chunks < 2^11
constexpr uint64_t SZ_MAX_LANE = FLUSH_ELEMS / 2;

__device__ __forceinline__ uint32_t band_key(uint32_t k, uint32_t) {
    return mad_u32(k, 0xFFFF0001u, 0xFFFF0000u);              // lo16: k, hi16: 0xFFFF - k (k <= 2046)
}

__device__ __noinline__ void halfz_rescan(int64_t* col, const uint4* seg, uint64_t seg_vecs, int hl, uint32_t& flags,
                                          uint32_t one) {
    for (uint64_t v = hl; v < seg_vecs; v += LPS) {            // every vector this lane summed
        const uint4 q = ldg_stream(seg + v);
        column_fix_special(col, q.x, q.y, flags, one);
        column_fix_special(col, q.z, q.w, flags, one);
    }
}

// K6z's per-segment epilogue over NK row groups of the band (NK = 1: straight-line code)
template <int NK>
__device__ __forceinline__ void halfz_epilogue(int64_t* wb, const SegOut& o, int64_t* su, uint64_t* sink, uint64_t ps,
                                               uint64_t pp, uint64_t nseg, uint64_t seg_len, uint32_t flags, int base,
                                               int dhi, int hl, int half) {
    __syncwarp();
    HalfSums d;
#pragma unroll
    for (int k = 0; k < KD; ++k) d.hs[k] = d.ls[k] = 0;
    // lane hl sums row base + hl + LPS k of its half's 16 columns, reading column hl ^ c at step c
    // (a permutation across the half: conflict-free). The columns are 128-B aligned, so the address
    // of column hl ^ c is one XOR of the lane's column-hl address. Rows above dhi hold zeros.
    const uint32_t sw = (uint32_t)__cvta_generic_to_shared(wb) + half * (LPS * 8) + hl * 8;
#pragma unroll
    for (int k = 0; k < NK; ++k) {
        const int row = base + hl + LPS * k;
        if (row <= dhi) {
            const uint32_t A = sw + (uint32_t)row * 256u;
#pragma unroll
            for (int c0 = 0; c0 < LPS; c0 += 4) {      // groups of 4 loads in flight (register budget)
                int64_t v[4];
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v[c]) : "r"(A ^ (uint32_t)((c0 + c) * 8)) : "memory");
#pragma unroll
                for (int c = 0; c < 4; ++c)   // the next segment starts from zero
                    asm volatile("st.shared.b64 [%0], %1;" :: "r"(A ^ (uint32_t)((c0 + c) * 8)), "l"(0ll) : "memory");
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    d.hs[k] += v[c] >> 32;
                    d.ls[k] += (int64_t)(uint32_t)v[c];
                }
            }
        }
    }
    __syncwarp();
    int64_t a[KD];
    half_digits<NK>(d, a, hl, base);
    uint32_t fl = flags;
#pragma unroll
    for (int off = LPS / 2; off > 0; off >>= 1) fl |= __shfl_xor_sync(FULL, fl, off, LPS);
    const bool mine = SEGS * pp + half < nseg;
    uint64_t* cp = o.canon ? (mine ? o.canon + ps * XSUM_CANON_LIMBS : sink) : nullptr;
    xsum_result r = finalize_half<NK>(a, fl, seg_len, cp, su, hl, half, base);
    if (hl == 0 && mine) o.write(ps, r);
}

#ifndef XS_SZ_WARPS
#define XS_SZ_WARPS 16    // one block of 16 warps per SM: 658 vs 626 G/s for two blocks of 8 (c5)
#endif
#ifndef XS_SZ_MINB
#define XS_SZ_MINB 1
#endif
constexpr int SZ_WARPS = XS_SZ_WARPS;
constexpr size_t SZ_SMEM = (size_t)SZ_WARPS * D * 32 * sizeof(int64_t);
#ifndef XS_SZ_COH
#define XS_SZ_COH 0       // development: coherent (non-.nc) input loads
#endif
__device__ __forceinline__ uint4 sz_load(const uint4* p) { return XS_SZ_COH ? ld_stream(p) : ldg_stream(p); }

template <int SZ_U, int SZ_NB>
__global__ void __launch_bounds__(SZ_WARPS * 32, XS_SZ_MINB)
k_segments_halfz(const double* __restrict__ x, uint64_t nseg, uint64_t seg_len, SegOut o, uint32_t one, uint32_t mone) {
    extern __shared__ __align__(128) int64_t winz[];           // 128-B aligned columns (the epilogue's XOR)
    __shared__ int64_t su[SZ_WARPS][SEGS][48];
    __shared__ uint64_t canon_sink[SZ_WARPS][XSUM_CANON_LIMBS];   // the odd last pair's idle half
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, hl = lane & (LPS - 1), half = lane / LPS;
    int64_t* col = winz + warp * (D * 32) + lane;
    const uint64_t nw = (uint64_t)gridDim.x * SZ_WARPS;
    const uint64_t npairs = (nseg + SEGS - 1) / SEGS;
    const uint64_t gw = (uint64_t)blockIdx.x * SZ_WARPS + warp;
    if (gw >= npairs) return;                                  // warp-uniform
    constexpr uint32_t SZ_TILE = LPS * SZ_U * 2;                // doubles per segment tile
    const uint32_t TPS = (uint32_t)(seg_len / SZ_TILE);
    const uint64_t seg_vecs = seg_len / 2;
    const uint4* xv = reinterpret_cast<const uint4*>(x);
#pragma unroll
    for (int j = 0; j < D; ++j) col[j * 32] = 0;
    auto seg_of = [&](uint64_t p) -> uint64_t {
        const uint64_t s = SEGS * p + half;
        return s < nseg ? s : SEGS * p;
    };
    constexpr uint32_t TV = LPS * SZ_U;
    const uint4* lp = xv + seg_of(gw) * seg_vecs + hl;
    uint64_t lpair = gw;
    uint32_t lt = 0;
    auto advance_load = [&]() {
        lp += SZ_NB * TV;
        lt += SZ_NB;
        if (lt == TPS) {
            lt = 0;
            lpair += nw;
            lp = xv + seg_of(lpair < npairs ? lpair : gw) * seg_vecs + hl;
        }
    };
    uint64_t pp = gw;
    uint32_t pt = 0, band = 0;
    uint4 buf[SZ_NB][SZ_U];
#pragma unroll
    for (int bb = 0; bb < SZ_NB; ++bb)
#pragma unroll
        for (int u = 0; u < SZ_U; ++u) buf[bb][u] = sz_load(lp + bb * TV + u * LPS);
    advance_load();
    while (pp < npairs) {
        const bool ld = lpair < npairs;
#pragma unroll
        for (int bb = 0; bb < SZ_NB; ++bb) {
#pragma unroll
            for (int u = 0; u < SZ_U; ++u) {
                Chunks a = decompose(buf[bb][u].x, buf[bb][u].y, one, mone);
                column_add(col, a, one);
                Chunks c = decompose(buf[bb][u].z, buf[bb][u].w, one, mone);
                column_add(col, c, one);
                band = __vmaxu2(__vmaxu2(band, band_key(a.spec, one)), band_key(c.spec, one));
            }
            if (ld) {
#pragma unroll
                for (int u = 0; u < SZ_U; ++u) buf[bb][u] = sz_load(lp + bb * TV + u * LPS);
            }
        }
        if (ld) advance_load();
        pt += SZ_NB;
#ifdef XS_EXP_SZ_NOEPI
        if (pt == TPS) { pt = 0; pp += nw; band = 0; continue; }   // diagnostic: WRONG sums
#endif
        if (pt == TPS) {                                       // both halves' segments complete
            const uint64_t ps = seg_of(pp);
            uint32_t flags = 0;
            if (__any_sync(FULL, (band & 0xFFFFu) >= 2046u)) {  // rare: cancel NaN/Inf patterns
                if ((band & 0xFFFFu) >= 2046u) halfz_rescan(col, xv + ps * seg_vecs, seg_vecs, hl, flags, one);
            }
#pragma unroll
            for (int off = LPS / 2; off > 0; off >>= 1) band = __vmaxu2(band, __shfl_xor_sync(FULL, band, off, LPS));
            const int kmax = (int)(band & 0xFFFFu), kmin = 0xFFFF - (int)(band >> 16);
            const int dlo = kmin / 52, dhi = kmax / 52 + 1;    // the digits this half's chunks touched
            const int base = o.canon ? 0 : dlo;
            int nk = (dhi + 2 - base + LPS - 1) / LPS;         // rows base .. dhi + 1 (the top carry)
            nk = max(nk, __shfl_xor_sync(FULL, nk, LPS));
            nk = o.canon || nk > KD ? KD : nk;
            if (nk == 1)                                       // warp-uniform
                halfz_epilogue<1>(winz + warp * (D * 32), o, su[warp][half], canon_sink[warp], ps, pp, nseg, seg_len,
                                  flags, base, dhi, hl, half);
            else if (LPS < 16 && nk == 2)                      // quarter warps: c5's band is two groups
                halfz_epilogue<2>(winz + warp * (D * 32), o, su[warp][half], canon_sink[warp], ps, pp, nseg, seg_len,
                                  flags, base, dhi, hl, half);
            else
                halfz_epilogue<KD>(winz + warp * (D * 32), o, su[warp][half], canon_sink[warp], ps, pp, nseg, seg_len,
                                   flags, base, dhi, hl, half);
            band = 0;
            pt = 0;
            pp += nw;
        }
    }
}

#ifndef XS_SH_Z
#define XS_SH_Z 1
#endif
bool segments_half_ok(const double* x, uint64_t seg_len) {
    if (((uintptr_t)x & 15) != 0) return false;
    if (XS_SH_Z && seg_len >= SZ_GRAN2 && seg_len % SZ_GRAN2 == 0 && seg_len / LPS <= SZ_MAX_LANE) return true;
    return seg_len >= SH_TILE && seg_len % ((uint64_t)SH_TILE * SH_NB) == 0 && seg_len / SH_TILE < (1u << 31);
}

cudaError_t sum_segments_half(const double* x, uint64_t nseg, uint64_t seg_len, const SegOut& o, int num_sms,
                              cudaStream_t s) {
    const uint64_t npairs = (nseg + SEGS - 1) / SEGS;          // groups of SEGS segments
    const uint64_t want = (npairs + SH_WARPS - 1) / SH_WARPS;
    const uint64_t cap = (uint64_t)num_sms * XS_SH_MINB;
    const unsigned g = (unsigned)(want < cap ? (want ? want : 1) : cap);
    const uint64_t wantz = (npairs + SZ_WARPS - 1) / SZ_WARPS;
    const uint64_t capz = (uint64_t)num_sms * XS_SZ_MINB;
    const unsigned gz = (unsigned)(wantz < capz ? (wantz ? wantz : 1) : capz);
    if (XS_SH_Z && seg_len / LPS <= SZ_MAX_LANE && seg_len % SZ_GRAN1 == 0) {
        static unsigned long long smem_z = 0;
        if (cudaError_t e = ensure_smem(k_segments_halfz<SZ_U1, SZ_NB1>, SZ_SMEM, smem_z)) return e;
        k_segments_halfz<SZ_U1, SZ_NB1><<<gz, SZ_WARPS * 32, SZ_SMEM, s>>>(x, nseg, seg_len, o, 1u, 0xFFFFFFFFu);
        note_launch();
        return cudaGetLastError();
    }
    if (XS_SH_Z && seg_len / LPS <= SZ_MAX_LANE && seg_len % SZ_GRAN2 == 0) {
        static unsigned long long smem_z2 = 0;
        if (cudaError_t e = ensure_smem(k_segments_halfz<SZ_U2, 2>, SZ_SMEM, smem_z2)) return e;
        k_segments_halfz<SZ_U2, 2><<<gz, SZ_WARPS * 32, SZ_SMEM, s>>>(x, nseg, seg_len, o, 1u, 0xFFFFFFFFu);
        note_launch();
        return cudaGetLastError();
    }
    static unsigned long long smem_set = 0;
    if (cudaError_t e = ensure_smem(k_segments_half, SH_SMEM, smem_set)) return e;
    k_segments_half<<<g, SH_WARPS * 32, SH_SMEM, s>>>(x, nseg, seg_len, o, 1u, 0xFFFFFFFFu);
    note_launch();
    return cudaGetLastError();
}

}  // namespace xs
