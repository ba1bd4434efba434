/* ORACLE — test infrastructure only.
 *
 * A plain, slow, obviously correct CPU exact summer for IEEE-754 binary64 (the
 * "oracle" of DESIGN.md). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it. It shares no code, header,
 * table or constant with the CUDA path in paper_1605_05436_b200/.
 *
 * What it computes (the plain definition the method reaches exactly):
 *   PAPER.md:449-463 (§2, fixed-point view): every partial sum is a fixed-point
 *   binary number, "we would have no errors in summing the numbers in X". Every
 *   finite binary64 is an integer multiple of 2^-1074, so A = sum_i x_i * 2^1074
 *   is an integer. We hold A in NLIMB = 34 little-endian 64-bit limbs, two's
 *   complement (2176 bits >= 1074 + 1024 + 63 + 1 sign bit, enough for n < 2^63).
 *
 *   Decoding follows IEEE 754 binary64 (reading R1: the paper's bias
 *   2^{E-2^{l-1}-1}, is off by two from IEEE; reading R2:
 *   subnormals are summed exactly, "we do not assume ... normalized",
 *   PAPER.md:155-158): x = (-1)^s * M * 2^(k-1074), M = m + [e!=0]*2^52,
 *   k = max(e,1) - 1.
 *
 *   Rounding: round-to-nearest, ties-to-even (reading R3), one of the
 *   faithful roundings of PAPER.md:172-179 and the "correctly rounded" result of
 *   §5. Overflow to +-Inf per IEEE (R11).
 *   Specials (paper silent, R10): NaN if any NaN or both +Inf and -Inf; else the Inf.
 *   Exact zero gives +0.0 (R9).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NLIMB 34

#define OF_NAN      1u   /* a NaN was summed */
#define OF_PINF     2u   /* +Inf was summed */
#define OF_NINF     4u   /* -Inf was summed */
#define OF_OVERFLOW 8u   /* finite exact sum rounds beyond DBL_MAX -> +-Inf */
#define OF_INEXACT  16u  /* rounded value != exact finite sum */
#define OF_OVERFLOW32 64u   /* binary32 rounding: finite exact sum rounds beyond FLT_MAX */
#define OF_INEXACT32 128u   /* binary32 rounding != exact finite sum */

typedef struct {
    double   value;
    int32_t  direction;  /* sign(value - exact) of the finite part, 0 when a special is returned */
    uint32_t flags;
    int32_t  msb_exp;    /* floor(log2|exact|), or INT32_MIN for zero */
    int32_t  sign;       /* 1 if exact < 0 */
    uint64_t count;
    uint64_t sig53;      /* unbounded-exponent RN-even rounding: |exact| ~ sig53 * 2^exp2 */
    int32_t  exp2;
    uint32_t value_f32;  /* bits of the RN-even binary32 rounding of the exact sum */
} oracle_result;

/* A += v * 2^(64*at), v an unsigned 64-bit value; carry ripples to the top limb. */
static void limbs_add_u64(uint64_t *A, int at, uint64_t v) {
    for (int L = at; L < NLIMB && v; ++L) {
        uint64_t s = A[L] + v;
        v = (s < v) ? 1 : 0;
        A[L] = s;
    }
}

/* Add x_i for i < n: positive terms into the magnitude P, negative terms into the
 * magnitude N (both non-negative 34-limb integers; A = P - N is formed at the end,
 * exact integer addition being associative). One element at a time. */
void oracle_accumulate(uint64_t *P, uint64_t *N, uint32_t *flags, const double *x, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t b;
        memcpy(&b, &x[i], 8);
        uint64_t s = b >> 63;
        uint64_t e = (b >> 52) & 0x7FF;
        uint64_t m = b & ((1ull << 52) - 1);
        if (e == 0x7FF) {                       /* specials: recorded, not summed */
            if (m) *flags |= OF_NAN;
            else   *flags |= s ? OF_NINF : OF_PINF;
            continue;
        }
        uint64_t M = m | ((e != 0) ? (1ull << 52) : 0);
        if (M == 0) continue;                    /* +-0 */
        unsigned k = (e != 0) ? (unsigned)(e - 1) : 0u;   /* |x| = M 2^(k-1074) */
        int L = (int)(k / 64);
        unsigned sh = k % 64;
        uint64_t lo = M << sh;
        uint64_t hi = sh ? (M >> (64 - sh)) : 0;
        uint64_t *T = s ? N : P;
        limbs_add_u64(T, L, lo);
        limbs_add_u64(T, L + 1, hi);
    }
}

/* binary32 inputs (IEEE 754 binary32, t = 23, l = 8): |x| = M 2^(k-149),
 * M = m + [e!=0] 2^23, k = max(e,1)-1; in units of 2^-1074 that is M 2^(k+925). */
void oracle_accumulate_f32(uint64_t *P, uint64_t *N, uint32_t *flags, const float *x, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t b;
        memcpy(&b, &x[i], 4);
        uint32_t s = b >> 31;
        uint32_t e = (b >> 23) & 0xFF;
        uint32_t m = b & 0x7FFFFF;
        if (e == 0xFF) {
            if (m) *flags |= OF_NAN;
            else   *flags |= s ? OF_NINF : OF_PINF;
            continue;
        }
        uint64_t M = m | ((e != 0) ? (1u << 23) : 0);
        if (M == 0) continue;
        unsigned k = ((e != 0) ? e - 1 : 0) + 925;      /* bit position in units of 2^-1074 */
        int L = (int)(k / 64);
        unsigned sh = k % 64;
        uint64_t lo = M << sh;
        uint64_t hi = sh ? (M >> (64 - sh)) : 0;
        uint64_t *T = s ? N : P;
        limbs_add_u64(T, L, lo);
        limbs_add_u64(T, L + 1, hi);
    }
}

/* 16-bit formats given as bit patterns: IEEE 754 binary16 (t = 10, l = 5) and bfloat16
 * (t = 7, l = 8), the paper's general format of t fraction bits and an l-bit exponent
 * (IEEE bias 2^(l-1)-1 per reading R1):
 *   |x| = M 2^(k + 1 - bias - t), M = m + [e!=0] 2^t, k = max(e,1) - 1,
 * i.e. M at bit position k + 1 - bias - t + 1074 in units of 2^-1074 (binary16: k + 1050,
 * bfloat16: k + 941). The all-ones exponent field is NaN (m != 0) or +-Inf. */
void oracle_accumulate_h16(uint64_t *P, uint64_t *N, uint32_t *flags, const uint16_t *x, uint64_t n,
                           int t, int l) {
    const uint32_t emask = (1u << l) - 1, mmask = (1u << t) - 1;
    const int bias = (1 << (l - 1)) - 1;
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t b = x[i];
        uint32_t s = b >> 15;
        uint32_t e = (b >> t) & emask;
        uint32_t m = b & mmask;
        if (e == emask) {
            if (m) *flags |= OF_NAN;
            else   *flags |= s ? OF_NINF : OF_PINF;
            continue;
        }
        uint64_t M = m | ((e != 0) ? (1u << t) : 0);
        if (M == 0) continue;
        unsigned k = (unsigned)(((e != 0) ? (int)e - 1 : 0) + 1 - bias - t + 1074);
        int L = (int)(k / 64);
        unsigned sh = k % 64;
        uint64_t lo = M << sh;
        uint64_t hi = sh ? (M >> (64 - sh)) : 0;
        uint64_t *T = s ? N : P;
        limbs_add_u64(T, L, lo);
        limbs_add_u64(T, L + 1, hi);
    }
}

/* A += B (limbwise with carry). */
void oracle_limbs_add(uint64_t *A, const uint64_t *B) {
    uint64_t c = 0;
    for (int L = 0; L < NLIMB; ++L) {
        uint64_t s = A[L] + B[L];
        uint64_t c1 = s < A[L];
        uint64_t t = s + c;
        uint64_t c2 = t < s;
        A[L] = t;
        c = c1 | c2;
    }
}

/* A -= B (limbwise with borrow, two's complement wrap). */
void oracle_limbs_sub(uint64_t *A, const uint64_t *B) {
    uint64_t br = 0;
    for (int L = 0; L < NLIMB; ++L) {
        uint64_t a = A[L];
        uint64_t d = a - B[L];
        uint64_t b1 = a < B[L];
        uint64_t t = d - br;
        uint64_t b2 = d < br;
        A[L] = t;
        br = b1 | b2;
    }
}

/* input formats of sum_threads */
#define FMT_F64 0
#define FMT_F32 1
#define FMT_F16 2   /* binary16 */
#define FMT_BF16 3  /* bfloat16 */

typedef struct {
    const void *x;
    uint64_t n;
    int fmt;
    uint64_t P[NLIMB], N[NLIMB];
    uint32_t flags;
} part_t;

static void *part_run(void *arg) {
    part_t *p = (part_t *)arg;
    switch (p->fmt) {
    case FMT_F32:  oracle_accumulate_f32(p->P, p->N, &p->flags, (const float *)p->x, p->n); break;
    case FMT_F16:  oracle_accumulate_h16(p->P, p->N, &p->flags, (const uint16_t *)p->x, p->n, 10, 5); break;
    case FMT_BF16: oracle_accumulate_h16(p->P, p->N, &p->flags, (const uint16_t *)p->x, p->n, 7, 8); break;
    default:       oracle_accumulate(p->P, p->N, &p->flags, (const double *)p->x, p->n); break;
    }
    return NULL;
}

static void sum_threads(uint64_t *A, uint32_t *flags, const void *x, uint64_t n, int nthreads, int fmt) {
    if (nthreads < 1) nthreads = 1;
    if ((uint64_t)nthreads > n / 65536 + 1) nthreads = (int)(n / 65536 + 1);
    part_t *parts = (part_t *)calloc((size_t)nthreads, sizeof(part_t));
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    uint64_t per = n / (uint64_t)nthreads, rem = n % (uint64_t)nthreads, off = 0;
    size_t esz = fmt == FMT_F64 ? 8 : (fmt == FMT_F32 ? 4 : 2);
    for (int t = 0; t < nthreads; ++t) {
        parts[t].x = (const char *)x + off * esz;
        parts[t].n = per + ((uint64_t)t < rem ? 1 : 0);
        parts[t].fmt = fmt;
        off += parts[t].n;
        pthread_create(&th[t], NULL, part_run, &parts[t]);
    }
    for (int t = 0; t < nthreads; ++t) {
        pthread_join(th[t], NULL);
        oracle_limbs_add(A, parts[t].P);
        oracle_limbs_sub(A, parts[t].N);
        *flags |= parts[t].flags;
    }
    free(parts); free(th);
}

/* Exact sum of x[0..n) ADDED TO (A, flags) (two's complement limbs), using nthreads host
 * threads over contiguous chunks. Callers zero A and flags for a fresh sum. */
void oracle_sum(uint64_t *A, uint32_t *flags, const double *x, uint64_t n, int nthreads) {
    sum_threads(A, flags, x, n, nthreads, FMT_F64);
}

/* Same for binary32 inputs. */
void oracle_sum_f32(uint64_t *A, uint32_t *flags, const float *x, uint64_t n, int nthreads) {
    sum_threads(A, flags, x, n, nthreads, FMT_F32);
}

/* Same for 16-bit bit patterns: bf16 = 0 -> binary16, bf16 = 1 -> bfloat16. */
void oracle_sum_h16(uint64_t *A, uint32_t *flags, const uint16_t *x, uint64_t n, int nthreads, int bf16) {
    sum_threads(A, flags, x, n, nthreads, bf16 ? FMT_BF16 : FMT_F16);
}

static int bitlen64(uint64_t v) { int b = 0; while (v) { ++b; v >>= 1; } return b; }

/* bit j of the magnitude a (limbs) */
static int bit_at(const uint64_t *a, long j) {
    if (j < 0 || j >= 64L * NLIMB) return 0;
    return (int)((a[j / 64] >> (j % 64)) & 1);
}

/* any bit below position j (exclusive) set? */
static int any_below(const uint64_t *a, long j) {
    if (j <= 0) return 0;
    long full = j / 64;
    for (long L = 0; L < full && L < NLIMB; ++L) if (a[L]) return 1;
    if (full < NLIMB && (j % 64)) {
        uint64_t mask = (1ull << (j % 64)) - 1;
        if (a[full] & mask) return 1;
    }
    return 0;
}

/* Round the exact integer A (units of 2^-1074, two's complement in 34 limbs) to binary64,
 * round-to-nearest ties-to-even, following SURVEY.md §8(c) "O1 step 8" literally. */
void oracle_round(const uint64_t *A, uint32_t flags_in, uint64_t count, oracle_result *r) {
    memset(r, 0, sizeof(*r));
    r->count = count;
    uint32_t flags = flags_in & (OF_NAN | OF_PINF | OF_NINF);
    int neg = (int)(A[NLIMB - 1] >> 63);
    uint64_t a[NLIMB];
    if (neg) {   /* a = -A */
        uint64_t c = 1;
        for (int L = 0; L < NLIMB; ++L) { uint64_t t = ~A[L] + c; c = (c && t == 0) ? 1 : 0; a[L] = t; }
    } else {
        memcpy(a, A, sizeof(a));
    }
    int top = -1;
    for (int L = NLIMB - 1; L >= 0; --L) if (a[L]) { top = L; break; }
    uint64_t bits;
    int direction = 0;
    if (top < 0) {                       /* exact zero -> +0.0 */
        bits = 0;
        r->msb_exp = INT32_MIN;
        r->sign = 0;
        r->sig53 = 0;
        r->exp2 = 0;
    } else {
        long p = 64L * top + bitlen64(a[top]) - 1;    /* index of leading 1 */
        r->msb_exp = (int32_t)(p - 1074);
        r->sign = neg;
        if (p <= 52) {                    /* |A| < 2^53: subnormal or min-normal, exact */
            bits = a[0];
            r->sig53 = a[0];
            r->exp2 = -1074;
        } else {
            long sh = p - 52;
            uint64_t q = 0;
            for (long j = p; j >= sh; --j) q = (q << 1) | (uint64_t)bit_at(a, j);
            int guard = bit_at(a, sh - 1);
            int sticky = any_below(a, sh - 1);
            int up = guard && (sticky || (q & 1));
            if (guard || sticky) direction = up ? 1 : -1;
            q += (uint64_t)up;
            if (q == (1ull << 53)) { q >>= 1; sh += 1; }
            r->sig53 = q;
            r->exp2 = (int32_t)(sh - 1074);
            long Eb = sh + 1;
            if (Eb >= 2047) {
                bits = 0x7FFull << 52;   /* overflow -> Inf */
                flags |= OF_OVERFLOW;
                direction = 1;
            } else {
                bits = ((uint64_t)Eb << 52) | (q - (1ull << 52));
            }
        }
        if (direction) flags |= OF_INEXACT;
        if (neg) { bits |= 1ull << 63; direction = -direction; }
    }
    /* binary32 rounding of the same exact value (t = 23, subnormal unit 2^-149 = bit 925) */
    uint32_t b32 = 0;
    if (top >= 0) {
        long p = 64L * top + bitlen64(a[top]) - 1;
        long sh = p - 23 > 925 ? p - 23 : 925;
        uint64_t q = 0;
        for (long j = p; j >= sh; --j) q = (q << 1) | (uint64_t)bit_at(a, j);
        int guard = bit_at(a, sh - 1);
        int sticky = any_below(a, sh - 1);
        int up = guard && (sticky || (q & 1));
        if (guard || sticky) flags |= OF_INEXACT32;
        q += (uint64_t)up;
        if (sh == 925) {
            b32 = (uint32_t)q;                   /* subnormal / smallest normals: bits = q (q <= 2^24) */
        } else {
            if (q == (1ull << 24)) { q >>= 1; sh += 1; }
            long Eb = sh - 925 + 1;
            if (Eb >= 255) { b32 = 0x7F800000u; flags |= OF_OVERFLOW32 | OF_INEXACT32; }
            else b32 = ((uint32_t)Eb << 23) | (uint32_t)(q - (1ull << 23));
        }
        if (neg) b32 |= 0x80000000u;            /* a negative sum that rounds to 0 gives -0.0f */
    }
    if ((flags & OF_NAN) || ((flags & OF_PINF) && (flags & OF_NINF))) b32 = 0x7FC00000u;
    else if (flags & OF_PINF) b32 = 0x7F800000u;
    else if (flags & OF_NINF) b32 = 0xFF800000u;
    r->value_f32 = b32;

    if ((flags & OF_NAN) || ((flags & OF_PINF) && (flags & OF_NINF))) {
        bits = 0x7FF8000000000000ull; direction = 0;
    } else if (flags & OF_PINF) {
        bits = 0x7FF0000000000000ull; direction = 0;
    } else if (flags & OF_NINF) {
        bits = 0xFFF0000000000000ull; direction = 0;
    }
    memcpy(&r->value, &bits, 8);
    r->direction = direction;
    r->flags = flags;
}

/* Segmented sums (the per-segment definition of BASELINE config 5 and SURVEY.md §8(f) f1): segment
 * s is x[off[s] .. off[s+1]) of format fmt (0 binary64, 1 binary32, 2 binary16, 3 bfloat16); each
 * segment is summed exactly on its own (oracle_accumulate*) and rounded by oracle_round. Outputs
 * per segment: bits64[s] (binary64 bits), bits32[s] (binary32 bits), flags[s], and, if canon is not
 * NULL, the 34-limb image at canon[34 s]. Segments are spread over nthreads threads (segment s on
 * thread s mod nthreads); nothing is shared between segments. */
typedef struct {
    const void *x;
    int fmt;
    const uint64_t *off;
    uint64_t nseg;
    int t, nt;
    uint64_t *bits64;
    uint32_t *bits32, *flags;
    uint64_t *canon;
} segs_t;

static void *segs_run(void *arg) {
    segs_t *a = (segs_t *)arg;
    size_t esz = a->fmt == FMT_F64 ? 8 : (a->fmt == FMT_F32 ? 4 : 2);
    for (uint64_t s = (uint64_t)a->t; s < a->nseg; s += (uint64_t)a->nt) {
        part_t p;
        memset(&p, 0, sizeof p);
        p.x = (const char *)a->x + a->off[s] * esz;
        p.n = a->off[s + 1] - a->off[s];
        p.fmt = a->fmt;
        part_run(&p);
        uint64_t A[NLIMB];
        memset(A, 0, sizeof A);
        oracle_limbs_add(A, p.P);
        oracle_limbs_sub(A, p.N);
        oracle_result r;
        oracle_round(A, p.flags, p.n, &r);
        memcpy(&a->bits64[s], &r.value, 8);
        a->bits32[s] = r.value_f32;
        a->flags[s] = r.flags;
        if (a->canon) memcpy(a->canon + s * NLIMB, A, sizeof A);
    }
    return NULL;
}

void oracle_sum_segments(const void *x, int fmt, const uint64_t *off, uint64_t nseg, uint64_t *bits64,
                         uint32_t *bits32, uint32_t *flags, uint64_t *canon, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if ((uint64_t)nthreads > nseg) nthreads = nseg ? (int)nseg : 1;
    segs_t *args = (segs_t *)calloc((size_t)nthreads, sizeof(segs_t));
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int t = 0; t < nthreads; ++t) {
        segs_t a = {x, fmt, off, nseg, t, nthreads, bits64, bits32, flags, canon};
        args[t] = a;
        pthread_create(&th[t], NULL, segs_run, &args[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(args); free(th);
}
