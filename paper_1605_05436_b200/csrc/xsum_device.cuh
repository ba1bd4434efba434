// Device building blocks of the superaccumulator reduction (sm_100a).
//
// Citations: PAPER.md line numbers of Goodrich & Eldawy (arXiv 1605.05436).
// Notation follows the paper: radix R = 2^w (w = 52 here, reading R5 in DESIGN.md),
// digits Y_j with value sum_j Y_j R^j (in units of 2^-1074),
// (alpha,beta)-regularized with alpha = beta = R-1.
#pragma once

#include <assert.h>
#include <stdint.h>

// XS_CHECKED=1 builds (tools/checked_build.py) assert every shared-memory digit index and the
// int64 headroom invariant on device: the pool's compute-sanitizer is unavailable, so the GPU
// test-suite is run against this build as the bounds/overflow check. 0 in the product.
#ifndef XS_CHECKED
#define XS_CHECKED 0
#endif
#if XS_CHECKED
#define XS_ASSERT(c) assert(c)
#else
#define XS_ASSERT(c) ((void)0)
#endif

#include "xsum.h"

namespace xs {

constexpr int W = XSUM_RADIX_BITS;          // 52
constexpr int D = XSUM_NDIGITS;             // 42 digits: 2184 bits >= 1074+1024+63
constexpr int64_t R = 1ll << W;
constexpr uint64_t MASK = (1ull << W) - 1;
constexpr unsigned FULL = 0xffffffffu;

// Summands a lane column may take between two regularizations. Each summand adds one
// chunk (|chunk| <= 2^52) to at most one position of each digit. A window holds at most
// FLUSH_ELEMS hot-loop summands plus <= 17 head/tail/leftover summands on top of a
// regularized residue |Y| <= 2^51 + 2^11:
// 2^51 + 2^11 + (2016 + 17) * 2^52 + 2^51 < 2^63, so neither the adds nor the balanced
// carry (y + R/2) can overflow int64. NaN/Inf bit patterns summed unchecked are cancelled
// after the window's regularization, in a fresh window of the same bound (re-derived in
// tests/test_host_logic.py). The paper's "reserved extra bit" becomes
// 11 bits of headroom per int64 digit here. 2016 is a multiple of 8 and 16 (whole tiles).
constexpr int FLUSH_ELEMS = 2016;

// Summand counts of merged states: each is <= 2^63-1, so a + b fits in u64; a total beyond
// 2^63-1 saturates and sets XSUM_F_CAPACITY (include/xsum.h).
constexpr uint64_t COUNT_MAX = 0x7FFFFFFFFFFFFFFFull;
__device__ __forceinline__ uint64_t count_add(uint64_t a, uint64_t b, uint32_t& fl) {
    uint64_t r = a + b;
    if (r > COUNT_MAX || r < a) {
        r = COUNT_MAX;
        fl |= XSUM_F_CAPACITY;
    }
    return r;
}

// ---------------------------------------------------------------------------------
// Step 2 of the PRAM algorithm: split x into O(1) components whose
// exponents are multiples of the radix exponent. For binary64 (IEEE, reading R1/R2):
// |x| = M 2^(k-1074), M = m + [e!=0] 2^52 < 2^53, k = max(e,1)-1 in [0, 2045].
// With i = k / 52 and o = k mod 52, sM 2^o (sM = +-M) is split at bit 52 into
//   c0 = (sM 2^o) mod 2^52  in [0, 2^52)      -> digit i
//   c1 = floor(sM 2^o / 2^52) in [-2^52, 2^52) -> digit i+1
// so that c0 R^i + c1 R^(i+1) = x 2^1074 exactly. Integer adds only (PAPER.md:654-668:
// integer digits with explicit overlap). All 32-bit halves, no FP instructions.
// ---------------------------------------------------------------------------------
struct Chunks {
    uint32_t i;      // digit index of c0
    uint32_t spec;   // 1 iff the exponent field is 0x7FF (NaN/Inf pattern), else 0
    int64_t c0, c1;
};

// Integer helpers pinned to the FMA pipe (IMAD / IMAD.HI / IMAD.WIDE): the decode is
// otherwise ALU-pipe bound (ncu: profiles/). `one` is a runtime 1 (a kernel argument) so
// that ptxas cannot fold x*one+y back into an ALU-pipe IADD3.
__device__ __forceinline__ uint32_t mulhi_u32(uint32_t a, uint32_t b) {
    uint32_t r; asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r;
}
__device__ __forceinline__ int32_t mulhi_s32(int32_t a, int32_t b) {
    int32_t r; asm("mul.hi.s32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r;
}
__device__ __forceinline__ uint32_t mad_u32(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r; asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c)); return r;
}
// mulhi(x, K52) = floor(x / 52) for 0 <= x <= 2047 (K52 = 20165 * 2^12; 52*20165 = 2^20 + 4,
// relative error 4/2^20 < 1/(52*2047); checked for every x in tests/test_host_logic.py).
constexpr uint32_t K52 = 20165u << 12;

// Per summand ~14 ALU-pipe ops and ~12 FMA-pipe issue slots (IMAD = 1, IMAD.HI = 2; measured
// sm_100 rates in tools/op_bench.cu, profiles/r01_microbench.txt), no IMAD.WIDE (1/8 rate): the
// constant divisions and the hidden-bit / sign assembly run as IMADs so that the ALU pipe is not
// the binding resource (an ALU-only decode measured 85% ALU busy and 640 vs 684 G/s).
__device__ __forceinline__ Chunks decompose(uint32_t lo, uint32_t hi, uint32_t one, uint32_t mone = 0xFFFFFFFFu) {
    Chunks c;
    uint32_t h = hi & 0x7FFFFFFFu;                        // |x| high word
    uint32_t e = h >> 20;                                 // biased exponent
    uint32_t ep = max(e, 1u);
    uint32_t k = mad_u32(ep, one, 0xFFFFFFFFu);           // ep - 1 (IMAD)
    uint32_t i = mulhi_u32(k, K52);                       // k / 52 (IMAD.HI)
    uint32_t o = mad_u32(i, (uint32_t)-52, k);            // k mod 52 (IMAD)
    uint32_t r = mad_u32(o, mone, 52u);                   // 52 - o (IMAD)
    uint32_t mh = mad_u32(k, 0xFFF00000u, h);             // hidden bit | top 20 fraction bits (IMAD)
    int32_t S = (int32_t)hi >> 31;                        // sign mask
    uint64_t onec = ((uint64_t)(mh ^ (uint32_t)S) << 32) | (lo ^ (uint32_t)S);
    int64_t sM = (int64_t)onec - (int64_t)S;              // +-M (IADD3 + IMAD.X)
    c.c0 = (int64_t)(((uint64_t)sM << o) & MASK);
    c.c1 = sM >> r;
    c.i = i;
    c.spec = k;                                           // k == 2046 only for NaN/Inf (max-tracked)
    return c;
}

// Tracking of NaN/Inf bit patterns summed unchecked in the hot loop: a per-lane fold that
// is cheap per summand and tested once per window.
__device__ __forceinline__ uint32_t spec_fold(uint32_t acc, const Chunks& c) { return max(acc, c.spec); }
__device__ __forceinline__ bool spec_hit(uint32_t acc) { return acc >= 2046u; }

// Add one summand's chunks into a lane column (digit j at col[j*32]): the "localized"
// add of PAPER.md:1043-1047 with carries deferred (PAPER.md:669-673 lazy carries).
// (plain IADD3/IMAD.X adds: the LDS -> add -> STS chain is latency-critical)
#ifndef XS_EXPERIMENT
#define XS_EXPERIMENT 0   // development-only diagnostic builds (tools/variants.py); 0 in the product
#endif
__device__ __forceinline__ void column_add(int64_t* col, const Chunks& c, uint32_t one) {
    (void)one;
#if XS_EXPERIMENT == 1      // diagnostic: no shared-memory traffic (decode + loads only; WRONG sums)
    col[0] ^= (c.c0 ^ c.c1) & (int64_t)(c.i == 1000u);
#elif XS_EXPERIMENT == 2    // diagnostic: RMW always on digits 0/1 (no data-dependent addressing)
    col[0] += c.c0;
    col[32] += c.c1 + (int64_t)c.i;
#else
    XS_ASSERT(c.i + 1 < (uint32_t)D - 1);            // chunks land in digits <= 40
    int64_t* p = col + c.i * 32u;
    // room for one more chunk (|c| <= 2^52) and the balanced carry's +R/2
    XS_ASSERT(p[0] > -0x7FE0000000000000ll && p[0] < 0x7FE0000000000000ll);
    XS_ASSERT(p[32] > -0x7FE0000000000000ll && p[32] < 0x7FE0000000000000ll);
    p[0] += c.c0;
    p[32] += c.c1;
#endif
}

// Flags of a NaN/Inf bit pattern (only called when e == 0x7FF).
__device__ __forceinline__ uint32_t special_flags(uint32_t lo, uint32_t hi) {
    if ((hi & 0xFFFFFu) | lo) return XSUM_F_NAN;
    return (hi >> 31) ? XSUM_F_NINF : XSUM_F_PINF;
}

// Checked add for the non-hot paths (head/tail elements): specials are flagged, not added.
__device__ __forceinline__ void column_add_checked(int64_t* col, uint32_t lo, uint32_t hi, uint32_t& flags,
                                                   uint32_t one) {
    Chunks c = decompose(lo, hi, one);
    if (spec_hit(c.spec)) { flags |= special_flags(lo, hi); return; }
    column_add(col, c, one);
}

// Undo the chunks the unchecked hot loop added for a NaN/Inf pattern (rare path):
// adding the chunks of the sign-flipped pattern cancels the value exactly.
__device__ __forceinline__ void column_fix_special(int64_t* col, uint32_t lo, uint32_t hi, uint32_t& flags,
                                                   uint32_t one) {
    if (((hi >> 20) & 0x7FFu) != 0x7FFu) return;
    flags |= special_flags(lo, hi);
    column_add(col, decompose(lo, hi ^ 0x80000000u, one), one);
}

// Input element traits: how a 16-byte vector splits into summands, and the non-hot paths.
template <typename T> struct Elem;

template <> struct Elem<double> {
    static constexpr int PER_VEC = 2;
    __device__ static __forceinline__ uint32_t fold(uint32_t acc, const Chunks& c) { return spec_fold(acc, c); }
    __device__ static __forceinline__ bool hit(uint32_t acc) { return spec_hit(acc); }
    __device__ static __forceinline__ void add_vec(int64_t* col, const uint4& v, uint32_t& nspec, uint32_t one,
                                                   uint32_t mone) {
        Chunks a = decompose(v.x, v.y, one, mone);
        nspec = fold(nspec, a);
        column_add(col, a, one);
        Chunks b = decompose(v.z, v.w, one, mone);
        nspec = fold(nspec, b);
        column_add(col, b, one);
    }
    __device__ static __forceinline__ void fix_vec(int64_t* col, const uint4& v, uint32_t& flags, uint32_t one) {
        column_fix_special(col, v.x, v.y, flags, one);
        column_fix_special(col, v.z, v.w, flags, one);
    }
    __device__ static __forceinline__ void add_vec_checked(int64_t* col, const uint4& v, uint32_t& flags,
                                                           uint32_t one) {
        column_add_checked(col, v.x, v.y, flags, one);
        column_add_checked(col, v.z, v.w, flags, one);
    }
    __device__ static __forceinline__ void add_one_checked(int64_t* col, const double* p, uint32_t& flags,
                                                           uint32_t one) {
        uint2 q;
        asm volatile("ld.global.v2.u32 {%0,%1}, [%2];" : "=r"(q.x), "=r"(q.y) : "l"(p));   // coherent: see ld_stream
        column_add_checked(col, q.x, q.y, flags, one);
    }
};

// ---------------------------------------------------------------------------------
// Regularization (PAPER.md:559-576 with the GSD idea of PAPER.md:522-525): each digit
// is split as Y_j = C_{j+1} R + r_j with a balanced remainder r_j in [-R/2, R/2) and
// S_j = r_j + C_j. Each output digit depends only on digits j and j-1 (carry-free).
// Input |Y_j| < 2^63 - 2^51; output |S_j| <= R/2 + 2^11 <= R-1. The top digit D-1 only
// ever receives carries (its magnitude is bounded by the value), so it
// is not split.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ int64_t balanced_carry(int64_t y) { return (y + (R >> 1)) >> W; }

__device__ __forceinline__ void regularize_column_inl(int64_t* col) {
    int64_t cin = 0;
#pragma unroll 6
    for (int j = 0; j < D - 1; ++j) {
        int64_t y = col[j * 32];
        XS_ASSERT(y > -0x7FF0000000000000ll && y < 0x7FF0000000000000ll);   // headroom kept
        int64_t c = balanced_carry(y);
        col[j * 32] = y - (c << W) + cin;
        cin = c;
    }
    col[(D - 1) * 32] += cin;
}

// Out-of-line copy for the rare paths (NaN/Inf compensation, leftovers).
__device__ __noinline__ static void regularize_column(int64_t* col) {
    int64_t cin = 0;
#pragma unroll 6
    for (int j = 0; j < D - 1; ++j) {
        int64_t y = col[j * 32];
        XS_ASSERT(y > -0x7FF0000000000000ll && y < 0x7FF0000000000000ll);   // headroom kept
        int64_t c = balanced_carry(y);
        col[j * 32] = y - (c << W) + cin;
        cin = c;
    }
    col[(D - 1) * 32] += cin;
}

// Digit-parallel regularization in a warp: lane l holds digit l (a0) and, for l < 10,
// digit l+32 (a1).
__device__ __forceinline__ void regularize_warp(int64_t& a0, int64_t& a1, int lane) {
    int64_t c0 = balanced_carry(a0);
    int64_t c1 = (lane + 32 < D - 1) ? balanced_carry(a1) : 0;
    int64_t in0 = __shfl_up_sync(FULL, c0, 1);
    int64_t in1 = __shfl_up_sync(FULL, c1, 1);
    int64_t c31 = __shfl_sync(FULL, c0, 31);
    if (lane == 0) { in0 = 0; in1 = c31; }
    a0 = a0 - (c0 << W) + in0;
    a1 = (lane + 32 < D) ? a1 - (c1 << W) + in1 : 0;
}

// Sum the 32 lane columns of a warp WITHOUT regularizing them first, into regularized
// digits (a0 = digit lane, a1 = digit lane+32). Each raw digit satisfies |Y| < 2^62, so it
// is split as Y = hi*2^32 + lo (lo unsigned 32-bit): the lane sums of lo (< 2^37) and hi
// (|.| < 2^35) cannot overflow; the balanced carry of D = HI*2^32 + LO is then
// c = (HI + ((LO + 2^51) >> 32)) >> 20 (exact floor), and the remainder
// r = (HI - c*2^20)*2^32 + LO. Output as regularize_warp.
struct LaneSums {          // per lane: digits lane and lane+32, each as (sum of hi words, sum of lo words)
    int64_t hs0, ls0, hs1, ls1;
};

__device__ __forceinline__ LaneSums raw_lane_sums(const int64_t* wb, int lane) {
    LaneSums t = {0, 0, 0, 0};
#pragma unroll 8
    for (int c = 0; c < 32; ++c) {
        int cc = (lane + c) & 31;                       // rotated: conflict-free columns
        int64_t v0 = wb[lane * 32 + cc];
        t.hs0 += v0 >> 32;
        t.ls0 += (int64_t)(uint32_t)v0;
        if (lane + 32 < D) {
            int64_t v1 = wb[(lane + 32) * 32 + cc];
            t.hs1 += v1 >> 32;
            t.ls1 += (int64_t)(uint32_t)v1;
        }
    }
    return t;
}

// Digits D_j = hs_j 2^32 + ls_j (|hs| < 2^40, |ls| < 2^50) -> regularized digits: balanced
// carry c = floor((D + 2^51) / 2^52) = (hs + ((ls + 2^51) >> 32)) >> 20 (exact floor since
// 0 <= ls + 2^51 < 2^52), remainder r = (hs - c 2^20) 2^32 + ls in [-2^51, 2^51).
__device__ __forceinline__ void sums_to_digits(const LaneSums& t, int64_t& a0, int64_t& a1, int lane) {
    auto split = [](int64_t hs, int64_t ls, int64_t& c, int64_t& r) {
        c = (hs + ((ls + (1ll << 51)) >> 32)) >> 20;
        r = (int64_t)((uint64_t)(hs - (c << 20)) << 32) + ls;
    };
    int64_t c0, r0, c1 = 0, r1 = 0;
    split(t.hs0, t.ls0, c0, r0);
    if (lane + 32 < D - 1) split(t.hs1, t.ls1, c1, r1);
    else if (lane + 32 == D - 1) { c1 = 0; r1 = (int64_t)((uint64_t)t.hs1 << 32) + t.ls1; }
    int64_t in0 = __shfl_up_sync(FULL, c0, 1), in1 = __shfl_up_sync(FULL, c1, 1);
    int64_t c31 = __shfl_sync(FULL, c0, 31);
    if (lane == 0) { in0 = 0; in1 = c31; }
    a0 = r0 + in0;
    a1 = (lane + 32 < D) ? r1 + in1 : 0;
}

// Sum the 32 lane columns of a warp WITHOUT regularizing them first, into regularized
// digits (a0 = digit lane, a1 = digit lane+32). Each raw digit is split as Y = hi 2^32 + lo
// (lo unsigned 32-bit): the lane sums of lo (< 2^37) and hi (|.| < 2^36) cannot overflow.
__device__ __forceinline__ void combine_raw_columns(const int64_t* wb, int64_t& a0, int64_t& a1, int lane) {
    sums_to_digits(raw_lane_sums(wb, lane), a0, a1, lane);
}

// ---------------------------------------------------------------------------------
// Lemma 1: sum of two (R-1,R-1)-regularized superaccumulators.
// P_j = Y_j + Z_j; C_{j+1} = 1 if P_j >= R-1, -1 if P_j <= -R+1, else 0 (reading R6);
// W_j = P_j - C_{j+1} R; S_j = W_j + C_j. Digit-parallel across the warp.
// The top digit (j = D-1) is never split (value bound).
// ---------------------------------------------------------------------------------
__device__ __forceinline__ int lemma1_carry(int64_t P) {
    return P >= R - 1 ? 1 : (P <= -(R - 1) ? -1 : 0);
}

__device__ __forceinline__ void lemma1_add(int64_t& a0, int64_t& a1, int64_t b0, int64_t b1, int lane) {
    int64_t P0 = a0 + b0, P1 = a1 + b1;
    int C0 = lemma1_carry(P0);
    int C1 = (lane + 32 < D - 1) ? lemma1_carry(P1) : 0;
    int64_t W0 = P0 - (int64_t)C0 * R, W1 = P1 - (int64_t)C1 * R;
    int in0 = __shfl_up_sync(FULL, C0, 1);
    int in1 = __shfl_up_sync(FULL, C1, 1);
    int c31 = __shfl_sync(FULL, C0, 31);
    if (lane == 0) { in0 = 0; in1 = c31; }
    a0 = W0 + in0;
    a1 = (lane + 32 < D) ? W1 + in1 : 0;
}

// ---------------------------------------------------------------------------------
// Steps 6-7 of the PRAM algorithm, one warp:
//  6. signed-carry propagation to the non-overlapping form by a parallel prefix over
//     carries in {-1,0} ("a simple lookup table based on whether the input carry bit is
//     -1, 0, or 1"): generate/propagate masks from two ballots and one
//     64-bit add (carry-lookahead), giving digits u_j in [0, R) of |A| (reading R4).
//  7. locate the most significant non-zero component, combine it with its neighbours and
//     round to nearest, ties to even, on the truncated bits (reading R3, R11).
// Input: regularized digits (|a| <= R-1), a0 = digit lane, a1 = digit lane+32.
// su: 64 int64 of shared scratch owned by this warp.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t extract_bits(const int64_t* su, int pos, int cnt) {
    // bits [pos, pos+cnt) (cnt <= 64, pos >= 0) of sum_j su[j] 2^(52 j), su[j] in [0, 2^52)
    uint64_t r = 0;
    int j0 = pos / 52;
    int j1 = (pos + cnt - 1) / 52;
    for (int j = j0; j <= j1 && j < D; ++j) {
        uint64_t v = (uint64_t)su[j];
        int sh = 52 * j - pos;
        if (sh >= 0) { if (sh < 64) r |= v << sh; }
        else r |= v >> (-sh);
    }
    return cnt >= 64 ? r : (r & ((1ull << cnt) - 1));
}

// Returns the result record in lane 0 (other lanes: unspecified); writes the canonical
// image (34 limbs) to `canon` if non-null.
__device__ __forceinline__ xsum_result finalize_warp_inl(int64_t a0, int64_t a1, uint32_t flags, uint64_t count,
                                                         uint64_t* canon, int64_t* su, int lane) {
    xsum_result r = {};
    const bool has1 = lane + 32 < D;
    uint64_t nz = (uint64_t)__ballot_sync(FULL, a0 != 0) | ((uint64_t)__ballot_sync(FULL, a1 != 0) << 32);
    int sign = 0;
    if (nz) {
        int msd = 63 - __clzll((long long)nz);
        int64_t top = __shfl_sync(FULL, msd < 32 ? a0 : a1, msd & 31);
        sign = top < 0;
    }
    if (sign) { a0 = -a0; a1 = -a1; }           // now sum > 0 (or zero)

    // split a = b R + r, r in [0,R), b in {-1,0}; t_j = r_j + b_{j-1} in [-1, R-1]
    int64_t b0 = a0 >> W, b1 = a1 >> W;
    int64_t r0 = a0 & (int64_t)MASK, r1 = a1 & (int64_t)MASK;
    if (lane + 32 == D - 1) { r1 = a1; b1 = 0; }    // top digit: not split
    int64_t in0 = __shfl_up_sync(FULL, b0, 1), in1 = __shfl_up_sync(FULL, b1, 1);
    int64_t b31 = __shfl_sync(FULL, b0, 31);
    if (lane == 0) { in0 = 0; in1 = b31; }
    int64_t t0 = r0 + in0, t1 = has1 ? r1 + in1 : 0;
    // borrow-lookahead: g_j = (t_j == -1), p_j = (t_j == 0); borrow_in = ((G|P) + G) ^ P
    uint64_t G = (uint64_t)__ballot_sync(FULL, t0 == -1) | ((uint64_t)__ballot_sync(FULL, has1 && t1 == -1) << 32);
    uint64_t P = (uint64_t)__ballot_sync(FULL, t0 == 0) | ((uint64_t)__ballot_sync(FULL, has1 && t1 == 0) << 32);
    uint64_t CI = ((G | P) + G) ^ P;
    int64_t u0 = (t0 - (int64_t)((CI >> lane) & 1)) & (int64_t)MASK;
    int64_t u1 = t1 - (int64_t)((CI >> (lane + 32)) & 1);
    if (lane + 32 < D - 1) u1 &= (int64_t)MASK;
    uint64_t nzu = (uint64_t)__ballot_sync(FULL, u0 != 0) | ((uint64_t)__ballot_sync(FULL, has1 && u1 != 0) << 32);

    // canonical image: 34 little-endian u64 limbs of A (two's complement)
    if (canon) {
        su[lane] = u0;
        if (has1) su[lane + 32] = u1;
        __syncwarp();
        uint64_t l0 = extract_bits(su, 64 * lane, 64);
        uint64_t l1 = (lane + 32 < XSUM_CANON_LIMBS) ? extract_bits(su, 64 * (lane + 32), 64) : 0;
        if (sign) {
            uint64_t z = (uint64_t)__ballot_sync(FULL, l0 != 0) | ((uint64_t)__ballot_sync(FULL, l1 != 0) << 32);
            int zl = z ? __ffsll((long long)z) - 1 : 64;     // lowest non-zero limb
            l0 = lane < zl ? 0 : (lane == zl ? (uint64_t)(-(int64_t)l0) : ~l0);
            l1 = lane + 32 < zl ? 0 : (lane + 32 == zl ? (uint64_t)(-(int64_t)l1) : ~l1);
        }
        canon[lane] = l0;
        if (lane + 32 < XSUM_CANON_LIMBS) canon[lane + 32] = l1;
    }

    // Step 7: lanes 0 and 1 round the same exact value in parallel, lane 0 to binary64
    // (t = 52, least subnormal 2^-1074 = bit 0, exponent field < 2047) and lane 1 to binary32
    // (t = 23, least subnormal 2^-149 = bit 925, exponent field < 255): one routine,
    // ties-to-even on the guard and sticky bits (reading R3).
    const bool is64 = lane == 0;
    const int prec = is64 ? 53 : 24, emin = is64 ? 0 : 925, emax = is64 ? 2047 : 255;
    uint64_t bits = 0;
    uint32_t rf = 0;                              // flags of this lane's rounding
    int dir = 0, msb = INT32_MIN, sh_out = 0;
    uint64_t q_out = 0;
    if (nzu) {                                    // warp-uniform
        // The guard bit lies at most prec+1 <= 54 bits below the leading bit, so the kept bits
        // and the guard bit sit in the three digits m, m-1, m-2 (m = top non-zero digit):
        // Wp = (d_m 2^104 + d_{m-1} 2^52 + d_{m-2}) >> 51 < 2^105 holds them (bit 0 of Wp =
        // bit 52m-53 of |A|); everything below Wp is sticky.
        const int m = 63 - __clzll((long long)nzu);
        auto digit = [&](int j) -> uint64_t {     // digit j (warp-uniform j), 0 for j < 0
            uint64_t v = (uint64_t)__shfl_sync(FULL, j >= 32 ? u1 : u0, j & 31);
            return j >= 0 ? v : 0;
        };
        const uint64_t dm = digit(m), dm1 = digit(m - 1), dm2 = digit(m - 2);
        if (lane < 2) {
            const int p = 52 * m + (63 - __clzll((long long)dm));   // leading bit of |A|
            msb = p - 1074;
            int sh = p - (prec - 1) > emin ? p - (prec - 1) : emin;
            const unsigned __int128 Wp = ((unsigned __int128)dm << 53) | ((unsigned __int128)dm1 << 1) | (dm2 >> 51);
            const int s = sh - 52 * m + 53;                         // >= 54 - prec >= 1
            uint64_t q = 0;
            int g = 0;
            bool sticky;                                            // any bit below the guard bit
            if (s < 128) {
                q = (uint64_t)(Wp >> s);
                g = (int)((uint64_t)(Wp >> (s - 1)) & 1);
                sticky = (Wp & (((unsigned __int128)1 << (s - 1)) - 1)) != 0;
            } else {
                sticky = Wp != 0;                                   // guard bit above Wp: 0
            }
            sticky = sticky || (dm2 & ((1ull << 51) - 1)) || (m >= 3 && (nzu & ((1ull << (m - 2)) - 1)));
            int up = g && (sticky || (q & 1));
            if (g || sticky) dir = up ? 1 : -1;
            q += (uint64_t)up;
            if (sh == emin) {
                bits = q;                             // subnormal / smallest normals: bits = q
            } else {
                if (q == (1ull << prec)) { q >>= 1; sh += 1; }
                int Eb = sh - emin + 1;
                if (Eb >= emax) { bits = (uint64_t)emax << (prec - 1); rf |= is64 ? XSUM_F_OVERFLOW : XSUM_F_OVERFLOW32; dir = 1; }
                else bits = ((uint64_t)Eb << (prec - 1)) | (q - (1ull << (prec - 1)));
            }
            q_out = q;
            sh_out = sh;
            if (dir) rf |= is64 ? XSUM_F_INEXACT : XSUM_F_INEXACT32;
            if (sign) { bits |= is64 ? (1ull << 63) : 0x80000000ull; dir = -dir; }   // -0.0f possible (R18)
        }
    }
    const uint64_t b32 = __shfl_sync(FULL, bits, 1);
    const uint32_t rf32 = __shfl_sync(FULL, rf, 1);
    if (lane == 0) {
        r.count = count;
        uint32_t fl = (flags & (XSUM_F_NAN | XSUM_F_PINF | XSUM_F_NINF | XSUM_F_MISMATCH | XSUM_F_PEER_TIMEOUT |
                                 XSUM_F_CAPACITY)) | rf | rf32;
        uint32_t v32 = (uint32_t)b32;
        if (!nzu) {                               // exact zero -> +0.0 (reading R9)
            r.msb_exp = INT32_MIN; r.sign = 0; r.sig53 = 0; r.exp2 = 0;
        } else {
            r.msb_exp = msb;
            r.sign = sign;
            r.sig53 = q_out;                      // unbounded-exponent rounding (before overflow)
            r.exp2 = sh_out - 1074;
        }
        if ((fl & XSUM_F_NAN) || ((fl & XSUM_F_PINF) && (fl & XSUM_F_NINF))) {
            bits = 0x7FF8000000000000ull; dir = 0; v32 = 0x7FC00000u;
        } else if (fl & XSUM_F_PINF) {
            bits = 0x7FF0000000000000ull; dir = 0; v32 = 0x7F800000u;
        } else if (fl & XSUM_F_NINF) {
            bits = 0xFFF0000000000000ull; dir = 0; v32 = 0xFF800000u;
        }
        r.value = __longlong_as_double((long long)bits);
        r.value_f32 = v32;
        r.direction = dir;
        r.flags = fl;
    }
    __syncwarp();
    return r;
}

// Out-of-line copy for the latency-insensitive callers (grid merge, finalize kernels).
__device__ __noinline__ static xsum_result finalize_warp(int64_t a0, int64_t a1, uint32_t flags, uint64_t count,
                                                         uint64_t* canon, int64_t* su, int lane) {
    return finalize_warp_inl(a0, a1, flags, count, canon, su, lane);
}

// The next segment of a warp: the next ticket (dynamic assignment) or cur + nw (static order).
__device__ __forceinline__ uint64_t seg_next(unsigned long long* ticket, uint64_t cur, uint64_t nw, int lane) {
    if (!ticket) return cur + nw;
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1ull);
    return (uint64_t)__shfl_sync(FULL, t, 0);
}

// 128-bit streaming load of two doubles as four 32-bit halves (no L1 allocation; 256-B L2
// prefetch: the best of the load flavours measured, profiles/r01_microbench.txt).
__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

// The same load without .nc, for kernels launched with programmatic dependent launch (the
// accumulate kernels K2/K2f/K2h): .nc declares the data read-only for the kernel's lifetime, and
// ptxas does schedule ld.global.nc above griddepcontrol.wait (the SASS of k_accumulate_f32b had its
// first LDG.CONSTANT tiles ahead of ACQBULK, and tests/test_gpu_api_r02.py's early-triggering
// producer caught the stale reads). With PDL the input may still be being written before the wait.
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ float ld_coherent(const float* p) {
    float v;
    asm volatile("ld.global.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint16_t ld_coherent(const uint16_t* p) {
    uint16_t v;
    asm volatile("ld.global.u16 %0, [%1];" : "=h"(v) : "l"(p));
    return v;
}

__device__ __forceinline__ uint2 ldg_one(const double* p) {
    uint2 v;
    asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}

}  // namespace xs
