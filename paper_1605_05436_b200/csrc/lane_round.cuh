// Per-lane (one thread) pieces shared by the kernels whose lanes own independent sums (K10
// strided reductions, K11 short segments): widening element loaders, canonicalization of one
// lane column and RN-even rounding from its top three digits, the canonical image.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "xsum_device.cuh"

namespace xs {

// Element loaders: every binary32 / binary16 / bfloat16 value is exactly a binary64 value, so
// the narrow formats are widened on load (cvt is exact, keeps subnormals, NaN and Inf) and
// summed by the binary64 decomposition.
template <int DT> struct StrLd;
template <> struct StrLd<XSUM_DT_F64> {
    using T = double;
    __device__ static __forceinline__ uint2 load(const T* p) {
        uint2 v;
        asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
        return v;
    }
};
__device__ __forceinline__ uint2 widen(float f) {
    const double d = (double)f;
    return make_uint2((uint32_t)__double2loint(d), (uint32_t)__double2hiint(d));
}
template <> struct StrLd<XSUM_DT_F32> {
    using T = float;
    __device__ static __forceinline__ uint2 load(const T* p) {
        uint32_t b;
        asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(b) : "l"(p));
        return widen(__uint_as_float(b));
    }
};
template <> struct StrLd<XSUM_DT_F16> {
    using T = uint16_t;
    __device__ static __forceinline__ uint2 load(const T* p) {
        unsigned short b;
        asm volatile("ld.global.nc.L1::no_allocate.b16 %0, [%1];" : "=h"(b) : "l"(p));
        return widen(__half2float(__ushort_as_half(b)));
    }
};
template <> struct StrLd<XSUM_DT_BF16> {
    using T = uint16_t;
    __device__ static __forceinline__ uint2 load(const T* p) {
        unsigned short b;
        asm volatile("ld.global.nc.L1::no_allocate.b16 %0, [%1];" : "=h"(b) : "l"(p));
        return widen(__uint_as_float((uint32_t)b << 16));
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

}  // namespace xs
