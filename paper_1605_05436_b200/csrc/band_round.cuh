// Per-slot (one segment per LPS lanes of a warp) regularization, carry-lookahead canonicalization
// and RN-even rounding of a segment's digits held in registers: lane hl of a slot holds digits
// base + hl + LPS k (k < NK, relative positions; all other digits zero). Shared by K6h / K6z (half
// warps, LPS = 16, segments_half.cu) and K6's values-only CSR epilogue (whole warps, LPS = 32).
// PAPER.md:559-576 (regularization), :777-795 (steps 6-7: signed-carry propagation and rounding).
#pragma once
#include "xsum_device.cuh"
#include "xsum_kernels.h"

namespace xs {

// Raw digit sums of a slot (hi / lo 32-bit words apart, as raw_lane_sums: no overflow).
template <int LPS>
struct SlotSums {
    static constexpr int KD = (D + LPS - 1) / LPS;
    int64_t hs[KD], ls[KD];
};

template <int LPS>
__device__ __forceinline__ uint32_t slot_bits(uint32_t ballot, int half) {
    if constexpr (LPS == 32) return ballot;
    else return (ballot >> (LPS * half)) & ((1u << LPS) - 1);
}

// Digits hl + LPS k of the slot's sum, regularized (balanced carry to the next digit; the top
// digit 41 is not split).
template <int LPS, int NK, int KD = (D + LPS - 1) / LPS>
__device__ __forceinline__ void slot_carry_in(const int64_t (&c)[KD], int64_t (&in)[KD], int hl) {
    // the carry into digit j comes from digit j-1: lane hl-1 of the same row group, or the
    // slot's last lane of the group below (for hl == 0)
#pragma unroll
    for (int k = 0; k < KD; ++k) {
        if (k >= NK) { in[k] = 0; continue; }
        const int64_t up = __shfl_up_sync(FULL, c[k], 1, LPS);
        const int64_t lo = k > 0 ? __shfl_sync(FULL, c[k > 0 ? k - 1 : 0], LPS - 1, LPS) : 0;
        in[k] = hl == 0 ? lo : up;
    }
}
// (base, NK: the slot's digits base + hl + LPS k for k < NK; the rest are zero)
template <int LPS, int NK, int KD = (D + LPS - 1) / LPS>
__device__ __forceinline__ void slot_digits(const SlotSums<LPS>& d, int64_t (&a)[KD], int hl, int base = 0) {
    int64_t c[KD], r[KD], in[KD];
#pragma unroll
    for (int k = 0; k < KD; ++k) {
        const int row = base + hl + LPS * k;
        if (k >= NK) {
            c[k] = 0;
            r[k] = 0;
        } else if (row < D - 1) {
            c[k] = (d.hs[k] + ((d.ls[k] + (1ll << 51)) >> 32)) >> 20;
            r[k] = (int64_t)((uint64_t)(d.hs[k] - (c[k] << 20)) << 32) + d.ls[k];
        } else if (row == D - 1) {
            c[k] = 0;
            r[k] = (int64_t)((uint64_t)d.hs[k] << 32) + d.ls[k];
        } else {
            c[k] = 0;
            r[k] = 0;
        }
    }
    slot_carry_in<LPS, NK>(c, in, hl);
#pragma unroll
    for (int k = 0; k < KD; ++k) a[k] = k < NK && base + hl + LPS * k < D ? r[k] + in[k] : 0;
}

// finalize_warp for a half warp: digits hl + 16k in a[k] (regularized); lane hl == 0 of each half
// returns the record (binary64 and binary32 roundings, RN-even).
// Positions are relative to the slot's base digit (bit j of a mask and digit_at(j): digit base + j);
// base > 0 or NK < KD need zero digits below base and above base + LPS NK (the banded kernel) and no
// canonical image (canon == nullptr unless base == 0 and NK == KD).
template <int LPS, int NK, int KD = (D + LPS - 1) / LPS>
__device__ __forceinline__ xsum_result slot_finalize(int64_t (&a)[KD], uint32_t flags, uint64_t count, uint64_t* canon,
                                                     int64_t* su, int hl, int half, int base = 0) {
    xsum_result res = {};
    auto valid = [&](int k) { return k < NK && base + hl + LPS * k < D; };
    auto mask = [&](auto pred) -> uint64_t {          // bit j: pred(k) of lane j % LPS, k = j / LPS (relative)
        uint64_t m = 0;
#pragma unroll
        for (int k = 0; k < KD; ++k)
            if (k < NK) m |= (uint64_t)slot_bits<LPS>(__ballot_sync(FULL, valid(k) && pred(k)), half) << (LPS * k);
        return m;
    };
    auto digit_at = [&](const int64_t (&v)[KD], int j) -> int64_t {   // relative digit j of this slot
        const int src = j & (LPS - 1), kk = j / LPS;
        int64_t out = 0;
#pragma unroll
        for (int k = 0; k < KD; ++k) {
            if (k >= NK) break;
            const int64_t w = __shfl_sync(FULL, v[k], src, LPS);
            if (k == kk) out = w;
        }
        return j < 0 ? 0 : out;
    };
    const uint64_t nz = mask([&](int k) { return a[k] != 0; });
    int sign = 0;
    {
        const int msd = nz ? 63 - __clzll((long long)nz) : 0;
        const int64_t top = digit_at(a, msd);
        sign = nz && top < 0;
    }
    if (sign) {
#pragma unroll
        for (int k = 0; k < KD; ++k) a[k] = -a[k];
    }
    int64_t b[KD], r[KD], t[KD], in[KD];
#pragma unroll
    for (int k = 0; k < KD; ++k) {
        b[k] = a[k] >> W;
        r[k] = a[k] & (int64_t)MASK;
        if (base + hl + LPS * k == D - 1) { r[k] = a[k]; b[k] = 0; }
    }
    slot_carry_in<LPS, NK>(b, in, hl);
#pragma unroll
    for (int k = 0; k < KD; ++k) t[k] = valid(k) ? r[k] + in[k] : 0;
    const uint64_t G = mask([&](int k) { return t[k] == -1; });
    const uint64_t P = mask([&](int k) { return t[k] == 0; });
    const uint64_t CI = ((G | P) + G) ^ P;
    int64_t u[KD];
#pragma unroll
    for (int k = 0; k < KD; ++k) {
        const int j = base + hl + LPS * k;
        u[k] = t[k] - (int64_t)((CI >> (hl + LPS * k)) & 1);
        if (j < D - 1) u[k] &= (int64_t)MASK;
        if (j >= D || k >= NK) u[k] = 0;
    }
    const uint64_t nzu = mask([&](int k) { return u[k] != 0; });

    if (canon) {                                   // rare: digits to shared memory, limbs per lane
#pragma unroll
        for (int k = 0; k < KD; ++k)
            if (hl + LPS * k < D) su[hl + LPS * k] = u[k];
        __syncwarp();
        for (int l = hl; l < XSUM_CANON_LIMBS; l += LPS) {
            uint64_t v = 0;
            const int pos = 64 * l, j0 = pos / 52, j1 = (pos + 63) / 52;
            for (int j = j0; j <= j1 && j < D; ++j) {
                const uint64_t dj = (uint64_t)su[j];
                const int sh = 52 * j - pos;
                if (sh >= 0) { if (sh < 64) v |= dj << sh; }
                else v |= dj >> (-sh);
            }
            canon[l] = v;                          // magnitude limbs; negated below if needed
        }
        __syncwarp();
        if (sign && hl == 0) {                     // two's complement: ~|A| + 1 (sequential, rare)
            uint64_t carry = 1;
            for (int l = 0; l < XSUM_CANON_LIMBS; ++l) {
                const uint64_t w = ~canon[l] + carry;
                carry = (carry && w == 0) ? 1 : 0;
                canon[l] = w;
            }
        }
        __syncwarp();
    }

    const bool is64 = hl == 0;
    const int prec = is64 ? 53 : 24, emin = is64 ? 0 : 925, emax = is64 ? 2047 : 255;
    uint64_t bits = 0;
    uint32_t rf = 0;
    int dir = 0, msb = INT32_MIN, sh_out = 0;
    uint64_t q_out = 0;
    const int m = nzu ? 63 - __clzll((long long)nzu) : 0;
    const uint64_t dm = (uint64_t)digit_at(u, m), dm1 = (uint64_t)digit_at(u, m - 1),
                   dm2 = (uint64_t)digit_at(u, m - 2);
    if (nzu && hl < 2) {
        const int p = 52 * (m + base) + (63 - __clzll((long long)dm));
        msb = p - 1074;
        int sh = p - (prec - 1) > emin ? p - (prec - 1) : emin;
        const unsigned __int128 Wp = ((unsigned __int128)dm << 53) | ((unsigned __int128)dm1 << 1) | (dm2 >> 51);
        const int s = sh - 52 * (m + base) + 53;
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
        sticky = sticky || (dm2 & ((1ull << 51) - 1)) || (m >= 3 && (nzu & ((1ull << (m - 2)) - 1)));
        const int up = g && (sticky || (q & 1));
        if (g || sticky) dir = up ? 1 : -1;
        q += (uint64_t)up;
        if (sh == emin) {
            bits = q;
        } else {
            if (q == (1ull << prec)) { q >>= 1; sh += 1; }
            const int Eb = sh - emin + 1;
            if (Eb >= emax) { bits = (uint64_t)emax << (prec - 1); rf |= is64 ? XSUM_F_OVERFLOW : XSUM_F_OVERFLOW32; dir = 1; }
            else bits = ((uint64_t)Eb << (prec - 1)) | (q - (1ull << (prec - 1)));
        }
        q_out = q;
        sh_out = sh;
        if (dir) rf |= is64 ? XSUM_F_INEXACT : XSUM_F_INEXACT32;
        if (sign) { bits |= is64 ? (1ull << 63) : 0x80000000ull; dir = -dir; }
    }
    const uint64_t b32 = __shfl_sync(FULL, bits, 1, LPS);
    const uint32_t rf32 = __shfl_sync(FULL, rf, 1, LPS);
    if (hl == 0) {
        res.count = count;
        const uint32_t fl = (flags & (XSUM_F_NAN | XSUM_F_PINF | XSUM_F_NINF)) | rf | rf32;
        uint32_t v32 = (uint32_t)b32;
        if (!nzu) {
            res.msb_exp = INT32_MIN; res.sign = 0; res.sig53 = 0; res.exp2 = 0;
        } else {
            res.msb_exp = msb; res.sign = sign; res.sig53 = q_out; res.exp2 = sh_out - 1074;
        }
        if ((fl & XSUM_F_NAN) || ((fl & XSUM_F_PINF) && (fl & XSUM_F_NINF))) {
            bits = 0x7FF8000000000000ull; dir = 0; v32 = 0x7FC00000u;
        } else if (fl & XSUM_F_PINF) {
            bits = 0x7FF0000000000000ull; dir = 0; v32 = 0x7F800000u;
        } else if (fl & XSUM_F_NINF) {
            bits = 0xFFF0000000000000ull; dir = 0; v32 = 0xFF800000u;
        }
        res.value = __longlong_as_double((long long)bits);
        res.value_f32 = v32;
        res.direction = dir;
        res.flags = fl;
    }
    return res;
}

}  // namespace xs
