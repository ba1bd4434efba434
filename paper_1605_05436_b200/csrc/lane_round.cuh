// Per-lane (one thread) pieces shared by the kernels whose lanes own independent sums (K10
// strided reductions, K11 short segments): the native decomposition of narrow-format elements,
// K10's element loaders, canonicalization of one lane column and RN-even rounding from its top
// three digits, the canonical image.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "xsum_device.cuh"
#include "xsum_kernels.h"

namespace xs {

// Native decomposition of a binary32 / binary16 / bfloat16 pattern (t fraction bits, l exponent
// bits, least subnormal at bit OFF of the 2^-1074 window: 925 / 1050 / 941): |x| = M 2^(k+OFF),
// M = m | [e != 0] 2^t, k = max(e,1) - 1 (reading R1), chunks of +-M 2^o at
// digit i = (k+OFF) / 52 as in decompose(); NaN/Inf patterns are marked (spec = 2046) and summed
// like finite ones, to be cancelled by fix_narrow on the rare path.
template <int TB, int LB, int OFF>
__device__ __forceinline__ Chunks dec_narrow(uint32_t b) {
    constexpr uint32_t EM = (1u << LB) - 1;
    const uint32_t e = (b >> TB) & EM;
    const uint32_t m = b & ((1u << TB) - 1);
    const uint32_t k = (e > 1u ? e : 1u) - 1u;
    const uint32_t sh = k + OFF;
    Chunks c;
    c.i = mulhi_u32(sh, K52);
    const uint32_t o = sh - 52u * c.i;
    const int64_t M = (int64_t)(m | ((e != 0u ? 1u : 0u) << TB));
    const int64_t sM = ((b >> (TB + LB)) & 1u) ? -M : M;
    c.c0 = (int64_t)(((uint64_t)sM << o) & MASK);
    c.c1 = sM >> (52u - o);
    c.spec = e == EM ? 2046u : k;
    return c;
}
template <int TB, int LB, int OFF>
__device__ __forceinline__ void fix_narrow(int64_t* col, uint32_t b, uint32_t& flags, uint32_t one) {
    constexpr uint32_t EM = (1u << LB) - 1;
    if (((b >> TB) & EM) != EM) return;
    flags |= (b & ((1u << TB) - 1)) ? XSUM_F_NAN : (((b >> (TB + LB)) & 1u) ? XSUM_F_NINF : XSUM_F_PINF);
    column_add(col, dec_narrow<TB, LB, OFF>(b ^ (1u << (TB + LB))), one);   // the negated pattern cancels it
}

// K10's loaders: raw(p) loads an element's bits, dec() decomposes them, fix() cancels a NaN/Inf
// pattern that was added unchecked (rescan).
template <int DT> struct StrLd;
template <> struct StrLd<XSUM_DT_F64> {
    using T = double;
    using R = uint2;
    __device__ static __forceinline__ R raw(const T* p) {
        uint2 v;
        asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
        return v;
    }
    __device__ static __forceinline__ Chunks dec(R r, uint32_t one, uint32_t mone) { return decompose(r.x, r.y, one, mone); }
    __device__ static __forceinline__ void fix(int64_t* col, R r, uint32_t& flags, uint32_t one) {
        column_fix_special(col, r.x, r.y, flags, one);
    }
};
template <> struct StrLd<XSUM_DT_F32> {
    using T = float;
    using R = uint32_t;
    __device__ static __forceinline__ R raw(const T* p) {
        uint32_t b;
        asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(b) : "l"(p));
        return b;
    }
    __device__ static __forceinline__ Chunks dec(R r, uint32_t, uint32_t) { return dec_narrow<23, 8, 925>(r); }
    __device__ static __forceinline__ void fix(int64_t* col, R r, uint32_t& flags, uint32_t one) {
        fix_narrow<23, 8, 925>(col, r, flags, one);
    }
};
template <> struct StrLd<XSUM_DT_F16> {
    using T = uint16_t;
    using R = uint32_t;
    __device__ static __forceinline__ R raw(const T* p) {
        unsigned short b;
        asm volatile("ld.global.nc.L1::no_allocate.b16 %0, [%1];" : "=h"(b) : "l"(p));
        return b;
    }
    __device__ static __forceinline__ Chunks dec(R r, uint32_t, uint32_t) { return dec_narrow<10, 5, 1050>(r); }
    __device__ static __forceinline__ void fix(int64_t* col, R r, uint32_t& flags, uint32_t one) {
        fix_narrow<10, 5, 1050>(col, r, flags, one);
    }
};
template <> struct StrLd<XSUM_DT_BF16> {
    using T = uint16_t;
    using R = uint32_t;
    __device__ static __forceinline__ R raw(const T* p) {
        unsigned short b;
        asm volatile("ld.global.nc.L1::no_allocate.b16 %0, [%1];" : "=h"(b) : "l"(p));
        return b;
    }
    __device__ static __forceinline__ Chunks dec(R r, uint32_t, uint32_t) { return dec_narrow<7, 8, 941>(r); }
    __device__ static __forceinline__ void fix(int64_t* col, R r, uint32_t& flags, uint32_t one) {
        fix_narrow<7, 8, 941>(col, r, flags, one);
    }
};

// One thread: regularized column (digit j at col[j*32]) -> sign and the canonical magnitude
// digits in place (borrow propagation); returns the top non-zero digit index m
// (-1 for an exact zero), the digits m, m-1, m-2 and whether anything below m-2 is non-zero.
struct LaneTop {
    int m;
    int sign;
    uint64_t dm, dm1, dm2;
    bool below;
};
// Digits outside [first, last] must be zero (callers that track the touched digit range pass it).
__device__ __forceinline__ LaneTop lane_canonical_top(int64_t* col, int first = 0, int last = D - 1) {
    LaneTop t = {-1, 0, 0, 0, 0, false};
    int top = last;
    while (top >= first && col[top * 32] == 0) --top;
    if (top < first) return t;
    t.sign = col[top * 32] < 0;
    int64_t br = 0;
    int lo = -1;                                   // lowest non-zero canonical digit
#pragma unroll 4
    for (int j = first; j <= top; ++j) {
        int64_t u = (t.sign ? -col[j * 32] : col[j * 32]) + br;
        if (j < D - 1) {
            br = u >> W;                           // u in [-R, R): borrow in {-1, 0}
            u &= (int64_t)MASK;
        }
        col[j * 32] = u;
        if (u != 0 && lo < 0) lo = j;
    }
    int m = top;
    while (m >= 0 && col[m * 32] == 0) --m;        // a borrow can clear the top digit
    t.m = m;
    t.dm = (uint64_t)col[m * 32];
    t.dm1 = m >= 1 ? (uint64_t)col[(m - 1) * 32] : 0;
    t.dm2 = m >= 2 ? (uint64_t)col[(m - 2) * 32] : 0;
    t.below = lo >= 0 && lo < m - 2;
    return t;
}

// A lane's RAW column digits [lo, hi] (|y| < 2^62, unregularized; digits outside are zero) to the
// LaneTop of their sum A, zeroing them, in one carry chain instead of regularize +
// lane_canonical_top (two read-write passes and scans; ncu r02: K11 issue-bound): t = y + c,
// d = t mod R, c = floor(t / R) gives the two's complement digits d_j of A (c settles to 0 or -1,
// the sign). For A >= 0 the magnitude digits are d_j; for A < 0 they are e_j = R-1-d_j above the
// lowest non-zero digit lz, R-d_lz at lz and 0 below (|A| = ~A + 1). So the chain only records the
// highest index with d != 0, the highest with d != R-1 and lz, and the window digits are read back.
template <int STRIDE = 32>
__device__ __forceinline__ LaneTop lane_top_chain(int64_t* col, int lo, int hi) {
    int64_t c = 0;
    int mpos = -1, mneg = -1, lz = -1;
    int j = lo;
    for (; j < D; ++j) {
        int64_t y = 0;
        if (j <= hi) y = col[j * STRIDE];
        else if (c == 0 || c == -1) break;             // the carry has settled: sign extension above
        const int64_t t = y + c;
        const uint64_t d = (uint64_t)t & MASK;
        c = t >> W;
        col[j * STRIDE] = (int64_t)d;
        mpos = d ? j : mpos;
        mneg = d != MASK ? j : mneg;
        lz = (lz < 0 && d) ? j : lz;
    }
    const int top = j - 1;                             // highest digit written
    LaneTop t = {-1, 0, 0, 0, 0, false};
    const bool neg = c < 0;
    if (neg && lz < 0) lz = top + 1;                   // all written digits 0: the first sign digit
    const int m = neg ? (mneg > lz ? mneg : lz) : mpos;
    if (m >= 0) {
        auto dig = [&](int k) -> uint64_t {            // magnitude digit k (k <= m)
            if (k < 0) return 0;
            // digits below lo were never written (zero); above top they are sign digits (R-1)
            const uint64_t d = k <= top ? (uint64_t)col[k * STRIDE] : MASK;
            if (!neg) return d;
            return k < lz ? 0 : (k == lz ? (uint64_t)R - d : MASK - d);
        };
        t.m = m;
        t.sign = neg;
        t.dm = dig(m);
        t.dm1 = dig(m - 1);
        t.dm2 = dig(m - 2);
        t.below = lz < m - 2;
    }
#pragma unroll 4
    for (int k = lo; k <= top; ++k) col[k * STRIDE] = 0;
    return t;
}

// RN-even rounding of the magnitude described by `t` to a format (prec, emin, emax as in
// finalize_warp: binary64 53 / 0 / 2047, binary32 24 / 925 / 255); the same three-digit window.
__device__ __forceinline__ uint64_t lane_round(const LaneTop& t, int prec, int emin, int emax, bool is64,
                                               uint32_t& rf) {
    if (t.m < 0) return 0;
    const int p = 52 * t.m + (63 - __clzll((long long)t.dm));
    int sh = p - (prec - 1) > emin ? p - (prec - 1) : emin;
    const unsigned __int128 Wp = ((unsigned __int128)t.dm << 53) | ((unsigned __int128)t.dm1 << 1) | (t.dm2 >> 51);
    const int s = sh - 52 * t.m + 53;
    uint64_t q = 0;
    int g = 0;
    bool sticky;
    if (s < 128) {
        q = (uint64_t)(Wp >> s);
        g = (int)((uint64_t)(Wp >> (s - 1)) & 1);
        sticky = (Wp & (((unsigned __int128)1 << (s - 1)) - 1)) != 0;
    } else {
        sticky = Wp != 0;
    }
    sticky = sticky || (t.dm2 & ((1ull << 51) - 1)) || t.below;
    const int up = g && (sticky || (q & 1));
    q += (uint64_t)up;
    uint64_t bits;
    if (sh == emin) {
        bits = q;
    } else {
        if (q == (1ull << prec)) { q >>= 1; sh += 1; }
        const int Eb = sh - emin + 1;
        if (Eb >= emax) {                          // +-Inf: never the exact value (finalize_warp's dir = 1)
            bits = (uint64_t)emax << (prec - 1);
            rf |= is64 ? (XSUM_F_OVERFLOW | XSUM_F_INEXACT) : (XSUM_F_OVERFLOW32 | XSUM_F_INEXACT32);
        } else {
            bits = ((uint64_t)Eb << (prec - 1)) | (q - (1ull << (prec - 1)));
        }
    }
    if (g || sticky) rf |= is64 ? XSUM_F_INEXACT : XSUM_F_INEXACT32;
    if (t.sign) bits |= is64 ? (1ull << 63) : 0x80000000ull;
    return bits;
}

// One thread: the canonical image (34 little-endian u64 limbs, two's complement) of the value
// whose magnitude digits (in [0, R), digit j at col[j*32], as left by lane_canonical_top) and
// sign are given; top = highest digit index to read (digits above are zero).
__device__ __forceinline__ void lane_canon_image(const int64_t* col, int top, int sign, uint64_t* out) {
    unsigned __int128 acc = 0;                    // pending bits, `have` of them valid
    int have = 0, limb = 0, j = 0;
    uint64_t carry = sign ? 1 : 0;                // two's complement: ~|A| + 1
    while (limb < XSUM_CANON_LIMBS) {
        while (have < 64 && j < D) {
            const uint64_t d = j <= top ? (uint64_t)col[j * 32] : 0;
            acc |= (unsigned __int128)d << have;
            have += 52;
            ++j;
        }
        uint64_t v = (uint64_t)acc;
        acc >>= 64;
        have = have > 64 ? have - 64 : 0;
        if (sign) {
            v = ~v;
            const uint64_t w = v + carry;
            carry = (carry && w == 0) ? 1 : 0;
            v = w;
        }
        out[limb++] = v;
    }
}

// (SegOut: xsum_kernels.h)
// the outputs of one segment from its roundings (b64 / b32 and their flags rf) and the NaN / Inf
// flags of its elements
__device__ __forceinline__ void lane_store_bits(uint64_t b64, uint32_t b32, uint32_t rf, uint32_t flags,
                                                const SegOut& o, uint64_t s) {
    const uint32_t fl = (flags & (XSUM_F_NAN | XSUM_F_PINF | XSUM_F_NINF)) | rf;
    if ((fl & XSUM_F_NAN) || ((fl & XSUM_F_PINF) && (fl & XSUM_F_NINF))) {
        b64 = 0x7FF8000000000000ull; b32 = 0x7FC00000u;
    } else if (fl & XSUM_F_PINF) {
        b64 = 0x7FF0000000000000ull; b32 = 0x7F800000u;
    } else if (fl & XSUM_F_NINF) {
        b64 = 0xFFF0000000000000ull; b32 = 0xFF800000u;
    }
    if (o.out) o.out[s] = __longlong_as_double((long long)b64);
    if (o.out32) o.out32[s] = __uint_as_float(b32);
    if (o.flags) o.flags[s] = fl;
}

// Values-only rounding of a lane's RAW digits [lo, hi] without the carry chain, when the top
// digits decide it (a Ziv-style test; round 2, for K11's short segments whose chain and rounding
// cost as much as their adds). T = y_hi R + y_(hi-1) (exact in 128 bits: |y_j| < len 2^52), or
// three digits when that is short, and the digits below add delta in (-len, len) units of T's
// last digit (|sum_{j<k} y_j R^j| < len R^k).
// With |T| >= 2^62 the sign and binade of A = (T + delta) R^(hi-1) are T's unless T mod 2^s lies
// within len of a multiple of 2^(s-1), s the rounding position (>= 10 here), and away from those
// points RN-even(A) = RN-even of any value within delta of T: the result is T's rounding and it is
// inexact. Without flags (need_flags false) only the midpoints are excluded: next to a multiple of
// 2^s the value is T's rounding as well, only its exactness is unknown (a gap of ~100 binades
// under a segment's largest element put 2% of c5s16's segments, and 44% of its warps, on the chain).
// Returns false (the caller runs the exact chain) when the test fails or hi < 1.
__device__ __forceinline__ bool lane_fast_round(const int64_t* col, int lo, int hi, int64_t len, bool want64,
                                                bool want32, bool need_flags, uint64_t& b64, uint32_t& b32,
                                                uint32_t& rf) {
    if (hi < 1 || hi < lo) return false;
    const int64_t yh = col[hi * 32], yl = hi - 1 >= lo ? col[(hi - 1) * 32] : 0;
    __int128 T = (__int128)yh * (__int128)R + (__int128)yl;
    int base = 52 * (hi - 1);
    // a short top (|T| < 2^74: the largest terms' upper chunks are small) takes the next digit too,
    // so that the rounding position sits far above delta and the test fails only ~2^-15 of the
    // time - a warp runs the chain if ANY lane needs it (|T R| < 2^126 + 2^56: still exact)
    const __int128 lim = (__int128)1 << 74;
    if (T < lim && T > -lim && hi >= 2 && hi - 2 >= lo) {
        T = T * (__int128)R + (__int128)col[(hi - 2) * 32];
        base -= 52;
    }
    const bool neg = T < 0;
    const unsigned __int128 mag = neg ? (unsigned __int128)(-T) : (unsigned __int128)T;
    const uint64_t mh = (uint64_t)(mag >> 64);
    if (!mh && ((uint64_t)mag >> 62) == 0) return false;           // |T| < 2^62
    const int pT = mh ? 127 - __clzll((long long)mh) : 63 - __clzll((long long)(uint64_t)mag);
    // the value test below needs 2 len < 2^(s-2) with s >= pT - 52: pT >= 57 + log2(len) (len <= 16:
    // any |T| >= 2^62; K11's rows of up to 256: 2^65)
    if (pT < 57 + (32 - __clz((int)(len - 1 > 0 ? len - 1 : 1)))) return false;
    const unsigned __int128 dl = (unsigned __int128)len;
    bool ok = true;
    uint32_t r = 0;
    auto one = [&](int prec, int emin, int emax, bool is64) -> uint64_t {
        const int P = pT + base;                                   // msb of |A| (binade fixed by the test)
        int sh = P - (prec - 1) > emin ? P - (prec - 1) : emin;    // lsb kept (absolute)
        const int sp = sh - base;                                  // ... in units of T: >= 10
        unsigned __int128 q, rem, half;
        if (sp >= 128) {                                           // |A| < 2^(sh-1): rounds to zero
            // (mag < 2^127 <= 2^(sp-1); the bound was 120 until round 2, which sent a three-digit T of
            // 2^119..2^126 with a binary32 rounding position 120..127 digits up into this branch
            // against a wrong half of 2^119: a sum of ~2^-276 rounded to the smallest subnormal)
            q = 0; rem = mag; half = (unsigned __int128)1 << 127;
        } else {
            q = mag >> sp;
            rem = mag & (((unsigned __int128)1 << sp) - 1);
            half = (unsigned __int128)1 << (sp - 1);
        }
        // near a midpoint the tail decides the value; near a representable value (rem within dl of
        // 0 or of 2 half) the value is decided - every point within 2 dl << half rounds to it, in the
        // lower binade too (dl < 2^(sp-2)) - and only INEXACT needs the tail: decided unless the
        // caller wants the flags
        if ((rem + dl > half && rem < half + dl) || (need_flags && (rem < dl || (sp < 128 && rem + dl > 2 * half)))) {
            ok = false;
            return 0;
        }
        uint64_t qq = (uint64_t)q + (rem > half ? 1u : 0u);
        uint64_t bits;
        if (sh == emin) {
            bits = qq;
        } else {
            if (qq == (1ull << prec)) { qq >>= 1; sh += 1; }
            const int Eb = sh - emin + 1;
            if (Eb >= emax) {
                bits = (uint64_t)emax << (prec - 1);
                r |= is64 ? XSUM_F_OVERFLOW : XSUM_F_OVERFLOW32;
            } else {
                bits = ((uint64_t)Eb << (prec - 1)) | (qq - (1ull << (prec - 1)));
            }
        }
        r |= is64 ? XSUM_F_INEXACT : XSUM_F_INEXACT32;
        if (neg) bits |= is64 ? (1ull << 63) : 0x80000000ull;
        return bits;
    };
    const uint64_t f64 = want64 ? one(53, 0, 2047, true) : 0;
    const uint32_t f32 = want32 ? (uint32_t)one(24, 925, 255, false) : 0;
    if (!ok) return false;
    b64 = f64;
    b32 = f32;
    rf |= r;
    return true;
}

// the outputs from a segment's canonical top (col: its canonical digits, read only for the image)
__device__ __forceinline__ void lane_store_top(const LaneTop& t, const int64_t* col, uint32_t flags, const SegOut& o,
                                               uint64_t s) {
    uint32_t rf = 0;
    // the binary32 rounding only when its value or the flags (which carry its bits) are wanted
    const bool want32 = o.out32 || o.flags;
    uint64_t b64 = (o.out || o.flags) ? lane_round(t, 53, 0, 2047, true, rf) : 0;
    uint32_t b32 = want32 ? (uint32_t)lane_round(t, 24, 925, 255, false, rf) : 0;
    const uint32_t fl = (flags & (XSUM_F_NAN | XSUM_F_PINF | XSUM_F_NINF)) | rf;
    if ((fl & XSUM_F_NAN) || ((fl & XSUM_F_PINF) && (fl & XSUM_F_NINF))) {
        b64 = 0x7FF8000000000000ull; b32 = 0x7FC00000u;
    } else if (fl & XSUM_F_PINF) {
        b64 = 0x7FF0000000000000ull; b32 = 0x7F800000u;
    } else if (fl & XSUM_F_NINF) {
        b64 = 0xFFF0000000000000ull; b32 = 0xFF800000u;
    }
    if (o.out) o.out[s] = __longlong_as_double((long long)b64);
    if (o.out32) o.out32[s] = __uint_as_float(b32);
    if (o.flags) o.flags[s] = fl;
    if (o.canon) lane_canon_image(col, t.m, t.sign, o.canon + s * XSUM_CANON_LIMBS);
}

}  // namespace xs
