// Decoding of 16-bit summands into exponent-group bins (binary16 / bfloat16), shared by the
// whole-array kernel K7 (accumulate_h16.cu) and the 16-bit segments kernel (segments_small.cu).
// See accumulate_h16.cu for the method and its citations.
#pragma once

#include "xsum_device.cuh"

namespace xs {

template <int T_, int L_, int SB_, int FLUSH_, int BASE_>
struct H16Fmt {
    static constexpr int t = T_;                          // fraction bits
    static constexpr int l = L_;                          // exponent bits
    static constexpr int SB = SB_;                        // exponent group = 2^SB consecutive exponents
    // q = max(e,1) + 1 in [2, 2^l - 1] for finite values, 2^l for NaN/Inf: group g = q >> SB,
    // offset o = q mod 2^SB; finite groups 0..NGF-1, the special group NGF.
    static constexpr int NGF = ((1 << l) - 1) / (1 << SB) + 1;
    static constexpr int NBIN = 2 * (NGF + 1);           // bin = 2 g + sign
    static constexpr int NBIN64 = 2 * NGF;                // finite bins only
    static constexpr int FLUSH = FLUSH_;                  // adds per window: FLUSH * max(M 2^o) < 2^32
    static constexpr int BASE = BASE_;                    // window bit position of k = 0 (units 2^-1074)
    // bin g holds sum M 2^o with M 2^k = (M 2^o) 2^(g 2^SB - 2): position BASE - 2 + g 2^SB
    static constexpr int pos(int g) { return BASE - 2 + g * (1 << SB); }
};
// Groups of 8 exponents for both formats: binary16 M <= 2047, o <= 7: 16383 * 2047 * 2^7 < 2^32
// (4 finite groups); bfloat16 M <= 255, o <= 7: 131071 * 255 * 2^7 < 2^32 (32 finite groups; the
// windows are long enough that emptying the bins is rare). Window bit positions: binary16
// k + 1050, bfloat16 k + 941.
using FmtF16 = H16Fmt<10, 5, 3, 16383, 1050>;
using FmtBF16 = H16Fmt<7, 8, 3, 131071, 941>;
// Segments empty their bins at every segment's end, so fewer bins beat longer windows there:
// bfloat16 groups of 16 exponents (17 groups; 511 * 255 * 2^15 < 2^32).
using FmtBF16Seg = H16Fmt<7, 8, 4, 511, 941>;
// The quarter-warp segments kernel empties its bins once per 16 steps of 32 elements per lane: the
// longest window that still fits, 514 * 255 * 2^15 < 2^32, covers one 4096-element segment.
using FmtBF16Q = H16Fmt<7, 8, 4, 514, 941>;
// a window of FLUSH adds of the largest M 2^o cannot wrap an unsigned 32-bit bin
template <class F>
constexpr bool flush_fits() {
    return (unsigned long long)F::FLUSH * ((2ull << F::t) - 1) * (1ull << ((1 << F::SB) - 1)) < (1ull << 32);
}
static_assert(flush_fits<FmtF16>() && flush_fits<FmtBF16>() && flush_fits<FmtBF16Seg>() && flush_fits<FmtBF16Q>(),
              "bin window too long");

// One summand (checked paths): h = |x| bit pattern (15 bits), s = sign bit; bins = this lane's
// bin column (bin b at word b*32).
template <class F>
__device__ __forceinline__ void h16_add(uint32_t* bins, uint32_t h, uint32_t s) {
    const uint32_t q = max((h >> F::t) + 1u, 2u);                          // max(e,1) + 1
    const uint32_t M = (h + (2u << F::t)) - q * (1u << F::t);              // m + [e!=0] 2^t
    const uint32_t o = q & ((1u << F::SB) - 1u);
    const uint32_t b = ((q >> F::SB) << 1) | s;
    XS_ASSERT(b < (uint32_t)F::NBIN);
    bins[b * 32u] += M << o;
}

__device__ __forceinline__ uint32_t vmax_u16x2(uint32_t a, uint32_t b) {
    uint32_t r; asm("max.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r;
}

__device__ __forceinline__ void bin_add(uint32_t saddr, uint32_t v) {
#ifdef XS_H16_LDSTS
    uint32_t o;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(o) : "r"(saddr) : "memory");
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(saddr), "r"(o + v) : "memory");
#else
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(saddr), "r"(v) : "memory");   // fire and forget
#endif
}

__device__ __forceinline__ uint32_t madhi_u32(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r; asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c)); return r;
}

// The two summands of a 32-bit word (little-endian: element 2i in the low half), decoded with
// the exponent work done once for both halves in 16-bit lanes (VIMNMX.U16x2, and IMADs / LOP3s
// whose per-half results cannot carry into the other half): per half q = max(e,1)+1 < 2^16,
// M = h + 2^(t+1) - q 2^t in [0, 2^(t+1)), bin byte offset (2 g + s) 128 < 2^16. The work is
// split between the ALU pipe (shifts, masks, min/max) and the FMA pipe (IMAD / IMAD.HI with
// the opaque `one` / `mone`), which ncu showed as the binding resource (ALU 93% busy in a plain
// version). `sbase` is the shared address of this lane's bin 0 (bin b at sbase + 128 b),
// `sbase2` = sbase * (2^16 + 1) mod 2^32.
template <class F>
__device__ __forceinline__ void h16_add_word(uint32_t sbase, uint32_t sbase2, uint32_t w, uint32_t one,
                                             uint32_t mone) {
    constexpr uint32_t t = F::t, SB = F::SB;
    constexpr uint32_t EM2 = ((1u << F::l) - 1u) * 0x00010001u;
    const uint32_t e2 = (w >> t) & EM2;                                       // exponent fields
    const uint32_t ep2 = vmax_u16x2(e2, 0x00010001u);                         // max(e,1)
    const uint32_t q2 = mad_u32(ep2, one, 0x00010001u);                       // + 1
    const uint32_t h2 = w & 0x7FFF7FFFu;                                      // |x| patterns
    const uint32_t M2 = mad_u32(ep2, 0u - (1u << t), mad_u32(h2, one, (1u << t) * 0x00010001u));  // M
    const uint32_t o2 = q2 & (((1u << SB) - 1u) * 0x00010001u);               // q mod 2^SB
    const uint32_t g2 = mad_u32(o2, mone, q2);                                // 2^SB g
    const uint32_t s2 = madhi_u32(mad_u32(h2, mone, w), 1u << 24, 0u);        // 128 s  (sign bits >> 8)
    const uint32_t a2 = mad_u32(g2, 1u << (8 - SB), s2);                      // (2 g + s) 128
    XS_ASSERT((a2 & 0xFFFFu) < (uint32_t)F::NBIN * 128u && (a2 >> 16) < (uint32_t)F::NBIN * 128u);
    const uint32_t Mh = M2 >> 16, oh = o2 >> 16;
    const uint32_t Ml = mad_u32(Mh, 0xFFFF0000u, M2);
    uint32_t vl;                      // Ml << o_lo: the wrap-mode funnel shift uses o2 mod 32 = o_lo
    asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(vl) : "r"(0u), "r"(Ml), "r"(o2));
    const uint32_t addr_hi = sbase + (a2 >> 16);
    const uint32_t addr_lo = mad_u32(addr_hi, 0xFFFF0000u, mad_u32(a2, one, sbase2));   // sbase + (a2 & 0xFFFF)
    bin_add(addr_lo, vl);
    bin_add(addr_hi, Mh << oh);
}

template <class F>
__device__ __forceinline__ uint32_t h16_special_flags(uint32_t b16) {
    if (((b16 >> F::t) & ((1u << F::l) - 1u)) != (1u << F::l) - 1u) return 0;
    if (b16 & ((1u << F::t) - 1u)) return XSUM_F_NAN;
    return (b16 >> 15) ? XSUM_F_NINF : XSUM_F_PINF;
}

// The bins are emptied into a narrow per-lane digit column holding only the digits the format
// reaches: row r is digit COL0 + r. A u32 bin (< 2^32) at bit position pos(g) spans <= 2 digits;
// COLS leaves room above for the carries of 2^63 summands; per flush a digit takes at most
// CHUNKS chunks (< 2^52 each), so REG_FLUSHES flushes fit the int64 headroom before the column
// must be regularized.
template <class F>
struct H16Col {
    static constexpr int COL0 = F::pos(0) / 52;
    static constexpr int COLS = F::pos(F::NGF - 1) / 52 + 2 - COL0 + 4;
    static constexpr int CHUNKS = 2 * ((52 + 84) / (1 << F::SB) + 1);
    static constexpr int REG_FLUSHES = 2000 / CHUNKS >= 64 ? 64 : (2000 / CHUNKS >= 32 ? 32 : 16);
};
static_assert(H16Col<FmtBF16>::REG_FLUSHES * H16Col<FmtBF16>::CHUNKS < 2048 &&
              H16Col<FmtBF16Seg>::REG_FLUSHES * H16Col<FmtBF16Seg>::CHUNKS < 2048 &&
              H16Col<FmtF16>::REG_FLUSHES * H16Col<FmtF16>::CHUNKS < 2048, "column headroom");

// Empty the finite u32 bins into the narrow column; returns true if this lane's NaN/Inf group
// was non-empty (and clears it: NaN/Inf are never summed).
template <class F>
__device__ __forceinline__ bool h16_flush_col(uint32_t* bins, int64_t* col) {
    using C = H16Col<F>;
#pragma unroll
    for (int j = 0; j < F::NBIN64; ++j) {
        const int P = F::pos(j >> 1), i = P / W - C::COL0, o = P % W;
        const uint64_t V = bins[j * 32];
        bins[j * 32] = 0;
        const int64_t c0 = (int64_t)((V << o) & MASK);
        const int64_t c1 = (int64_t)(V >> (W - o));                 // V 2^o < 2^84: two digits
        XS_ASSERT(i >= 0 && i + 1 < C::COLS - 1);
        if (j & 1) {
            col[i * 32] -= c0;
            col[(i + 1) * 32] -= c1;
        } else {
            col[i * 32] += c0;
            col[(i + 1) * 32] += c1;
        }
    }
    const uint32_t sp = bins[F::NBIN64 * 32] | bins[(F::NBIN64 + 1) * 32];
    bins[F::NBIN64 * 32] = 0;
    bins[(F::NBIN64 + 1) * 32] = 0;
    return sp != 0;
}

template <class F>
__device__ __forceinline__ void h16_col_regularize(int64_t* col) {
    constexpr int COLS = H16Col<F>::COLS;
    int64_t cin = 0;
#pragma unroll
    for (int j = 0; j < COLS - 1; ++j) {
        const int64_t y = col[j * 32];
        const int64_t c = balanced_carry(y);
        col[j * 32] = y - (c << W) + cin;
        cin = c;
    }
    col[(COLS - 1) * 32] += cin;
}

// A warp's narrow columns (wb: rows of 32 lanes) combined into the digit-parallel form: lane j
// returns digit j (all rows lie below digit 32). Row r is summed by lane r as hi/lo 32-bit halves
// (raw digits |Y| < 2^63), balanced carries are split off (the top row takes carries only) and
// move one row up.
template <class F>
__device__ __forceinline__ int64_t h16_col_combine(const int64_t* wb, int lane) {
    using C = H16Col<F>;
    static_assert(C::COL0 + C::COLS <= 32, "narrow column above digit 31");
    int64_t hs = 0, ls = 0;
    if (lane < C::COLS) {
#pragma unroll 8
        for (int c = 0; c < 32; ++c) {
            const int64_t v = wb[lane * 32 + ((lane + c) & 31)];
            hs += v >> 32;
            ls += (int64_t)(uint32_t)v;
        }
    }
    int64_t cr = 0, rr = (int64_t)((uint64_t)hs << 32) + ls;
    if (lane < C::COLS - 1) {
        cr = (hs + ((ls + (1ll << 51)) >> 32)) >> 20;
        rr = (int64_t)((uint64_t)(hs - (cr << 20)) << 32) + ls;
    }
    int64_t cin = __shfl_up_sync(FULL, cr, 1);
    if (lane == 0) cin = 0;
    const int64_t row = lane < C::COLS ? rr + cin : 0;
    const int64_t d = __shfl_sync(FULL, row, (lane - C::COL0) & 31);
    return (lane >= C::COL0 && lane < C::COL0 + C::COLS) ? d : 0;
}

}  // namespace xs
