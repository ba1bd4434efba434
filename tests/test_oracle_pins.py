"""Pins of the oracle (O1 = oracle/xsum_oracle.c, O2 = oracle/pytwin.py) against
things other than itself: hand-derived golden cases, exact rational brute force
(Fraction(float) is exact; float(Fraction) is CPython's correctly rounded int
division), math.fsum (Shewchuk, correctly rounded), invariants the problem fixes
(permutation, x + (-x) = 0, 2^1023 + 1 - 2^1023 = 1, the set-equality zero-sum
family of PAPER.md:812-839), the faithful-rounding bracket of PAPER.md:172-179,
and Lemma 1 exhaustively at R = 8.
"""
from __future__ import annotations

import math
import os
import random
import re
import struct
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import pytwin

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "rounding_edges.txt")


def f2b(x: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def b2f(b: int) -> float:
    return struct.unpack("<d", struct.pack("<Q", b))[0]


def load_golden():
    cases = []
    with open(GOLDEN) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            name, ins, out, direction, cite = [p.strip() for p in line.split("|")]
            xs = [b2f(int(h, 16)) for h in ins.split(",") if h.strip()]
            cases.append((name, xs, int(out, 16), int(direction), cite))
    return cases


GOLDEN_CASES = load_golden()


def exact_fraction(xs) -> Fraction:
    return sum((Fraction(x) for x in xs), Fraction(0))


def test_golden_file_has_citations():
    assert len(GOLDEN_CASES) >= 20
    for name, _, _, _, cite in GOLDEN_CASES:
        assert re.search(r"PAPER\.md:\d+|SPEC\.md:\d+|\bR\d+\b|north_star", cite), name


def test_golden_hex_literals_mean_what_they_say():
    # the hex inputs in the golden file are the doubles named in the derivations
    assert f2b(1e308) == 0x7FE1CCF385EBC8A0
    assert f2b(math.pi) == 0x400921FB54442D18
    assert f2b(2.0 ** -53) == 0x3CA0000000000000
    assert f2b(2.0 ** 970) == 0x7C90000000000000
    assert f2b(2.0 ** 1000) == 0x7E70000000000000
    assert f2b(2.0 ** -1000) == 0x0170000000000000
    assert f2b(5e-324) == 1
    assert f2b(2.0 ** 53) == 0x4340000000000000


@pytest.mark.parametrize("case", GOLDEN_CASES, ids=[c[0] for c in GOLDEN_CASES])
def test_golden_o1(case):
    name, xs, out_bits, direction, _ = case
    r, _ = oracle.exact_sum(np.array(xs, dtype=np.float64))
    assert r.bits == out_bits, f"{name}: {r.bits:016x} != {out_bits:016x}"
    assert r.direction == direction


@pytest.mark.parametrize("case", GOLDEN_CASES, ids=[c[0] for c in GOLDEN_CASES])
def test_golden_o2(case):
    name, xs, out_bits, direction, _ = case
    v, d, _, _ = pytwin.exact_sum(xs)
    assert f2b(v) == out_bits, name
    assert d == direction


def _random_double(rng: random.Random) -> float:
    """Finite doubles over the whole range incl. subnormals, zeros, boundary exponents."""
    kind = rng.random()
    if kind < 0.1:
        e = 0                                   # subnormal / zero
    elif kind < 0.2:
        e = rng.choice([1, 2, 1022, 1023, 1024, 2045, 2046])
    else:
        e = rng.randint(1, 2046)
    m = rng.getrandbits(52) if rng.random() < 0.9 else rng.choice([0, 1, (1 << 52) - 1])
    s = rng.getrandbits(1)
    return b2f((s << 63) | (e << 52) | m)


def _random_set(rng: random.Random, n: int) -> list[float]:
    mode = rng.random()
    if mode < 0.3:  # narrow exponent band -> many ties and cancellations
        e0 = rng.randint(1, 2040)
        xs = [b2f((rng.getrandbits(1) << 63) | (rng.randint(e0, e0 + 5) << 52) | rng.getrandbits(52))
              for _ in range(n)]
    elif mode < 0.45:  # add negations -> exact cancellation
        half = [_random_double(rng) for _ in range((n + 1) // 2)]
        xs = half + [-x for x in half[: n // 2]]
        rng.shuffle(xs)
    else:
        xs = [_random_double(rng) for _ in range(n)]
    return xs


def test_o1_vs_exact_fraction_bruteforce():
    """O1's image and rounding vs exact rationals (independent decoder: float.as_integer_ratio)."""
    rng = random.Random(1605)
    for trial in range(3000):
        xs = _random_set(rng, rng.randint(0, 9))
        r, limbs = oracle.exact_sum(np.array(xs, dtype=np.float64))
        S = exact_fraction(xs)
        A = S * (1 << 1074)
        assert A.denominator == 1
        assert oracle.limbs_to_int(limbs) == A.numerator, trial
        try:
            ref = float(S)
        except OverflowError:
            ref = math.inf if S > 0 else -math.inf
        if ref == 0.0:
            ref = 0.0
        assert r.bits == f2b(ref), (trial, xs)
        if S != 0 and not math.isinf(ref):
            assert r.direction == (Fraction(ref) > S) - (Fraction(ref) < S)


def test_o1_vs_fsum_in_range():
    """math.fsum is correctly rounded (Shewchuk) when no intermediate overflows."""
    rng = np.random.default_rng(7)
    for trial in range(200):
        n = int(rng.integers(1, 2000))
        e = rng.integers(-300, 300, size=n).astype(np.float64)
        x = rng.standard_normal(n) * np.exp2(e)
        if trial % 3 == 0:
            x = np.concatenate([x, -x[: n // 2]])
        r, _ = oracle.exact_sum(x)
        ref = math.fsum(x)
        if ref == 0.0:
            ref = 0.0
        assert r.bits == f2b(ref)


def test_o1_faithful_bracket():
    """result is the largest double <= S or the smallest double >= S."""
    rng = random.Random(11)
    for _ in range(2000):
        xs = _random_set(rng, rng.randint(1, 12))
        r, limbs = oracle.exact_sum(np.array(xs))
        if math.isinf(r.value):
            continue
        S = Fraction(oracle.limbs_to_int(limbs), 1 << 1074)
        v = Fraction(r.value)
        lo_f, hi_f = math.nextafter(r.value, -math.inf), math.nextafter(r.value, math.inf)
        assert math.isinf(lo_f) or Fraction(lo_f) < S
        assert math.isinf(hi_f) or S < Fraction(hi_f)
        if v != S:   # RN: within half an ulp
            ulp = Fraction(math.ulp(r.value))
            assert abs(v - S) <= ulp / 2


def test_o1_vs_o2_on_synth_prefixes():
    import synth
    for name in ("c1", "c2", "c4", "c5"):
        x = synth.gen.generate(name, 12345, 20000)
        r, limbs = oracle.exact_sum(x)
        v, d, fl, A = pytwin.exact_sum(x.tolist())
        assert [int(t) for t in limbs] == pytwin.limbs(A), name
        assert r.bits == f2b(v) and r.direction == d and r.flags == fl, name
    x = synth.gen.generate("c3", (1 << 28) - 5000, 10000, permute=False)  # pairs + tiny terms
    r, limbs = oracle.exact_sum(x)
    v, d, fl, A = pytwin.exact_sum(x.tolist())
    assert [int(t) for t in limbs] == pytwin.limbs(A)
    assert r.bits == f2b(v)


def test_o1_permutation_and_thread_invariance():
    rng = np.random.default_rng(3)
    bits = rng.integers(0, 2 ** 63, size=200_000, dtype=np.uint64) & np.uint64(0xFFEFFFFFFFFFFFFF)
    bits |= rng.integers(0, 2, size=bits.size, dtype=np.uint64) << np.uint64(63)
    x = bits.view(np.float64)
    r1, l1 = oracle.exact_sum(x, nthreads=1)
    for nt in (2, 3, 8):
        r, l = oracle.exact_sum(rng.permutation(x), nthreads=nt)
        assert (l == l1).all() and r.bits == r1.bits and r.flags == r1.flags


def test_o1_chunked_streaming_equals_whole():
    import synth
    x = synth.gen.generate("c2", 0, 100_000)
    whole = oracle.exact_sum(x)[1]
    acc = oracle.Accumulator()
    for a, b in [(0, 1), (1, 777), (777, 50_000), (50_000, 100_000)]:
        acc.add(x[a:b])
    assert (acc.limbs == whole).all() and acc.count == 100_000
    a1, a2 = oracle.Accumulator().add(x[:333]), oracle.Accumulator().add(x[333:])
    assert (a1.merge(a2).limbs == whole).all()


def test_x_plus_negx_is_plus_zero():
    import synth
    x = synth.gen.generate("c4", 0, 50_000)
    y = np.concatenate([x, -x[::-1]])
    r, limbs = oracle.exact_sum(y)
    assert r.bits == 0 and not limbs.any() and r.direction == 0


def test_set_equality_family():
    """PAPER.md:812-839 (Theorem 1 lower bound): -2^(tau c_i) and +2^(tau d_i) sum to zero
    iff the multisets C and D are equal; tau = smallest power of two > log n."""
    rng = random.Random(5)
    for trial in range(60):
        n = rng.randint(1, 300)
        tau = 1
        while tau <= math.log2(max(n, 2)):
            tau *= 2
        cmax = (2046 - 1) // tau                 # keep tau*c inside the binary64 exponent range
        C = [rng.randint(0, cmax) for _ in range(n)]
        D = list(C)
        rng.shuffle(D)
        equal = trial % 2 == 0
        if not equal:
            j = rng.randrange(n)
            D[j] = (D[j] + 1) % (cmax + 1)
        # exponents tau*c relative to 2^-1074 (unbiased exponent tau*c - 1074)
        xs = [-math.ldexp(1.0, tau * c - 1074) for c in C] + [math.ldexp(1.0, tau * d - 1074) for d in D]
        rng.shuffle(xs)
        r, limbs = oracle.exact_sum(np.array(xs))
        assert (not limbs.any()) == (sorted(C) == sorted(D)), trial
        if sorted(C) == sorted(D):
            assert r.bits == 0


def test_o2_rounding_matches_textbook_definition_on_boundaries():
    """O2 (library rounding) vs O1 (bit-level RN-even) on values straddling every
    rounding boundary shape: ties, near-ties, overflow threshold, subnormal/normal edge."""
    rng = random.Random(99)
    for _ in range(3000):
        p = rng.randint(0, 2160)
        sig = rng.getrandbits(min(p + 1, 60)) | (1 << min(p, 59))
        A = sig << max(0, p - 59)
        A += rng.choice([0, 1, -1, 1 << max(0, p - 53), (1 << max(0, p - 53)) - 1,
                         (1 << max(0, p - 53)) + 1])
        A *= rng.choice([1, -1])
        r = oracle.round_limbs(oracle.int_to_limbs(A), 0, 0)
        v, d, fl = pytwin.round_int(A)
        assert r.bits == f2b(v), hex(A)
        assert r.direction == d and r.flags == fl, hex(A)


def test_overflow_threshold_exact():
    """R11: RN overflows iff |S| >= 2^1024 - 2^970 (DBL_MAX + half ulp, tie to even 2^1024)."""
    t = (1 << (1024 + 1074)) - (1 << (970 + 1074))
    for A, inf in [(t, True), (t - 1, False), (-t, True), (-(t - 1), False)]:
        r = oracle.round_limbs(oracle.int_to_limbs(A), 0, 0)
        assert math.isinf(r.value) == inf
        assert bool(r.flags & oracle.F_OVERFLOW) == inf


def test_unbounded_rounding_fields():
    """sig53 * 2^exp2 is the RN-even rounding with an unbounded exponent (diagnostic for c4)."""
    A = ((1 << 53) - 1) << 2100     # beyond binary64 range
    r = oracle.round_limbs(oracle.int_to_limbs(A), 0, 0)
    assert math.isinf(r.value) and r.sig53 == (1 << 53) - 1 and r.exp2 == 2100 - 1074
    assert r.msb_exp == 2152 - 1074


# ---- Lemma 1, exhaustively at R = 8 (reading Q6 / DESIGN.md R6) ----

def lemma1_carry(P: int, R: int) -> int:
    if P >= R - 1:
        return 1
    if P <= -R + 1:
        return -1
    return 0


@pytest.mark.parametrize("R", [8, 16, 2 ** 5])
def test_lemma1_exhaustive(R):
    """For regularized Y, Z (digits in [-(R-1), R-1]) and any incoming carry C_i in {-1,0,1},
    S_i = P_i - C_{i+1} R + C_i stays in [-(R-1), R-1] (alpha = beta = R-1)."""
    a = R - 1
    for P in range(-2 * a, 2 * a + 1):
        C1 = lemma1_carry(P, R)
        W = P - C1 * R
        assert -(a - 1) <= W <= a - 1
        for Ci in (-1, 0, 1):
            assert -a <= W + Ci <= a


def test_lemma1_carry_free_addition_value_preserved():
    """Digit-local Lemma-1 addition of two regularized vectors preserves the value (R = 8)."""
    rng = random.Random(2)
    R, a = 8, 7
    for _ in range(2000):
        D = rng.randint(1, 8)
        Y = [rng.randint(-a, a) for _ in range(D)]
        Z = [rng.randint(-a, a) for _ in range(D)]
        P = [y + z for y, z in zip(Y, Z)] + [0]
        C = [0] + [lemma1_carry(P[i], R) for i in range(D)]          # C[i+1] from P[i]
        S = [P[i] - C[i + 1] * R + C[i] for i in range(D)] + [C[D]]
        val = lambda v: sum(d * R ** i for i, d in enumerate(v))
        assert val(S) == val(Y) + val(Z)
        assert all(-a <= s <= a for s in S)


# ---- binary32: inputs summed as binary32, and binary32 rounding ----

GOLDEN32 = os.path.join(os.path.dirname(__file__), "golden", "rounding_edges_f32.txt")


def load_golden32():
    cases = []
    with open(GOLDEN32) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            name, ins, out, cite = [p.strip() for p in line.split("|")]
            xs = [b2f(int(h, 16)) for h in ins.split(",") if h.strip()]
            cases.append((name, xs, int(out, 16), cite))
    return cases


GOLDEN32_CASES = load_golden32()


def test_golden32_hex_literals():
    assert f2b(float(np.float32(3.4028234663852886e38))) == 0x47EFFFFFE0000000
    assert f2b(2.0 ** -149) == 0x36A0000000000000 and f2b(2.0 ** 103) == 0x4660000000000000
    assert f2b(2.0 ** -54) == 0x3C90000000000000


@pytest.mark.parametrize("case", GOLDEN32_CASES, ids=[c[0] for c in GOLDEN32_CASES])
def test_golden32_o1_and_o2(case):
    name, xs, out32, cite = case
    assert re.search(r"PAPER\.md:\d+|\bR\d+\b", cite)
    r, limbs = oracle.exact_sum(np.array(xs, dtype=np.float64))
    assert r.bits_f32 == out32, f"{name}: {r.bits_f32:08x} != {out32:08x}"
    A, fl = pytwin.exact_int(xs)
    assert pytwin.round_int_f32(A, fl)[0] == out32, name


def _rand_f32_bits(rng, n):
    kind = rng.random()
    out = []
    for _ in range(n):
        if kind < 0.3:
            e = rng.randint(100, 106)
        else:
            e = rng.choice([0, 0, 1, 2, 126, 127, 253, 254]) if rng.random() < 0.3 else rng.randint(0, 254)
        out.append((rng.getrandbits(1) << 31) | (e << 23) | rng.getrandbits(23))
    return out


def test_o1_f32_inputs_vs_exact_rationals():
    """binary32 inputs: O1's exact image vs Fraction(float32) sums; its binary32 rounding vs
    the twin's search over neighbouring binary32 values with exact rational comparisons."""
    rng = random.Random(32)
    for trial in range(1500):
        bits = _rand_f32_bits(rng, rng.randint(0, 10))
        x = np.array(bits, dtype=np.uint32).view(np.float32)
        r, limbs = oracle.exact_sum(x)
        S = sum((Fraction(float(v)) for v in x), Fraction(0))
        assert oracle.limbs_to_int(limbs) == S * (1 << 1074), trial
        A, fl = pytwin.exact_int_f32(bits)
        assert A == oracle.limbs_to_int(limbs)
        b32, _ = pytwin.round_int_f32(A, fl)
        assert r.bits_f32 == b32, (trial, [hex(b) for b in bits])
        v, d, f, _ = pytwin.exact_sum([float(v) for v in x])
        assert r.bits == f2b(v) and r.flags == f


def test_o1_f32_rounding_on_boundaries():
    """binary32 rounding of integers straddling ties / overflow / subnormal edges (O1 bit-level
    algorithm vs the twin's rational search)."""
    rng = random.Random(33)
    for _ in range(3000):
        p = rng.randint(900, 1210)                      # binary32 range in units of 2^-1074
        A = (rng.getrandbits(30) | (1 << 29)) << max(0, p - 29)
        A += rng.choice([0, 1, -1, 1 << max(0, p - 24), (1 << max(0, p - 24)) - 1, 1 << max(0, p - 25)])
        A *= rng.choice([1, -1])
        r = oracle.round_limbs(oracle.int_to_limbs(A), 0, 0)
        b32, fl = pytwin.round_int_f32(A, 0)
        assert r.bits_f32 == b32, hex(A)
        assert (r.flags & (oracle.F_OVERFLOW32 | oracle.F_INEXACT32)) == fl


def test_f32_sum_equals_numpy_when_exactly_representable():
    """Sums of small integers as float32 are exact in any order: the binary32 rounding is the value."""
    rng = np.random.default_rng(4)
    for _ in range(50):
        x = rng.integers(-1000, 1000, size=1000).astype(np.float32)
        r, _ = oracle.exact_sum(x)
        expect = np.float32(int(x.astype(np.int64).sum()))
        assert r.bits_f32 == int(np.array([expect], dtype=np.float32).view(np.uint32)[0])


# ------------------------------------------------------------------------------------------
# 16-bit inputs (binary16 / bfloat16)
# ------------------------------------------------------------------------------------------
GOLDEN_H16 = os.path.join(os.path.dirname(__file__), "golden", "rounding_edges_h16.txt")


def load_golden_h16():
    cases = []
    with open(GOLDEN_H16) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            name, fmt, ins, o64, o32, cite = [p.strip() for p in line.split("|")]
            bits = np.array([int(h, 16) for h in ins.split(",")], dtype=np.uint16)
            cases.append((name, fmt, bits, int(o64, 16), int(o32, 16), cite))
    return cases


H16_CASES = load_golden_h16()


def h16_values(bits: np.ndarray, fmt: str) -> list:
    """Library decoders, independent of the oracle: numpy's binary16, and bfloat16 as the top
    half of a binary32 (its definition) decoded by numpy's float32."""
    bits = np.ascontiguousarray(bits, dtype=np.uint16)
    if fmt == "f16":
        return [float(v) for v in bits.view(np.float16)]
    return [float(v) for v in (bits.astype(np.uint32) << 16).view(np.float32)]


@pytest.mark.parametrize("case", H16_CASES, ids=[c[0] for c in H16_CASES])
def test_golden_h16(case):
    name, fmt, bits, o64, o32, cite = case
    assert re.search(r"PAPER\.md:\d+|\bR\d+\b", cite), name
    r, _ = oracle.exact_sum(bits, fmt=fmt)
    assert r.bits == o64, f"{name}: {r.bits:016x} != {o64:016x}"
    assert r.bits_f32 == o32, f"{name}: {r.bits_f32:08x} != {o32:08x}"
    # the hand-derived binary64 value agrees with the library decoders' exact sum
    vals = h16_values(bits, fmt)
    if all(math.isfinite(v) for v in vals):
        assert b2f(o64) == float(exact_fraction(vals))


def test_golden_h16_literals_mean_what_they_say():
    assert h16_values(np.array([0x3C00, 0x0001, 0x7BFF, 0x0400, 0x03FF], np.uint16), "f16") == \
        [1.0, 2.0 ** -24, 65504.0, 2.0 ** -14, 1023 * 2.0 ** -24]
    assert h16_values(np.array([0x3F80, 0x0001, 0x3380, 0x7F7F], np.uint16), "bf16") == \
        [1.0, 2.0 ** -133, 2.0 ** -24, (2 - 2.0 ** -7) * 2.0 ** 127]


@pytest.mark.parametrize("fmt", ["f16", "bf16"])
def test_h16_random_patterns_vs_rationals(fmt):
    # random bit patterns over the whole format (all exponents, subnormals, both signs; the
    # specials are dropped here and covered by the golden cases)
    rng = np.random.default_rng(16 if fmt == "f16" else 17)
    emask = 0x7C00 if fmt == "f16" else 0x7F80
    for trial in range(300):
        n = int(rng.integers(1, 60))
        bits = rng.integers(0, 1 << 16, size=n, dtype=np.uint32).astype(np.uint16)
        bits = bits[(bits & emask) != emask]
        vals = h16_values(bits, fmt)
        S = exact_fraction(vals)
        r, limbs = oracle.exact_sum(bits, fmt=fmt)
        assert oracle.limbs_to_int(limbs) == S * (1 << 1074)
        assert r.value == float(S) and (r.value != 0.0 or r.bits == 0)
        # binary32 rounding vs the twin's independent rational search
        b32, _ = pytwin.round_int_f32(int(S * (1 << 1074)))
        assert r.bits_f32 == b32


@pytest.mark.parametrize("fmt", ["f16", "bf16"])
def test_h16_o1_matches_o2_and_specials(fmt):
    rng = np.random.default_rng(5)
    bits = rng.integers(0, 1 << 16, size=20000, dtype=np.uint32).astype(np.uint16)
    r, limbs = oracle.exact_sum(bits, fmt=fmt, nthreads=3)
    A, flags = pytwin.exact_int_h16(bits, fmt)
    assert oracle.limbs_to_int(limbs) == A
    assert (r.flags & 7) == flags
    # chunking / threading invariance and permutation invariance
    r2, limbs2 = oracle.exact_sum(bits[::-1].copy(), fmt=fmt, nthreads=1)
    assert (limbs2 == limbs).all() and r2.bits == r.bits


def test_h16_all_binary16_finite_values_sum_to_zero():
    # every finite binary16 appears with both signs: the exact sum is 0 (+0.0, R9), while the
    # positive half alone is sum over e, m of the format's values (closed form below)
    allb = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    fin = allb[(allb & 0x7C00) != 0x7C00]
    r, limbs = oracle.exact_sum(fin, fmt="f16")
    assert r.bits == 0 and not limbs.any()
    pos = fin[fin < 0x8000]
    # closed form: subnormals sum_{m<1024} m 2^-24 + normals sum_{e=1..30} sum_m (1024+m) 2^(e-25)
    sub = Fraction(sum(range(1024)), 1 << 24)
    nor = sum(Fraction(sum(range(1024, 2048)) * 2 ** e, 1 << 25) for e in range(1, 31))
    _, lp = oracle.exact_sum(pos, fmt="f16")
    assert oracle.limbs_to_int(lp) == (sub + nor) * (1 << 1074)


# ------------------------------------------------------------------------------------------
# segmented sums (oracle.sum_segments: the per-segment definition of config 5 / f1)
# ------------------------------------------------------------------------------------------
def test_sum_segments_vs_o2_every_format():
    """Each segment of oracle.sum_segments against the independent Python twin O2 (exact Python
    ints, library rounding): ragged CSR bounds with empty segments, specials, every format."""
    import synth
    x64 = synth.gen.generate("c2", 5, 6000)
    x64[17] = np.inf
    x64[4000] = np.nan
    lens = [0, 1, 2, 3, 0, 17, 100, 1000, 0, 2000, 2877]
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    assert off[-1] == x64.size
    b64, b32, fl, cn = oracle.sum_segments(x64, off, canon=True, nthreads=3)
    for s in range(len(lens)):
        seg = x64[int(off[s]):int(off[s + 1])]
        A, f = pytwin.exact_int(seg)
        v, _, f2 = pytwin.round_int(A, f)
        assert int(b64[s]) == pytwin.bits_of(v) and int(fl[s]) & 0xFF & ~0xC0 == f2 & ~0xC0
        assert [int(c) for c in cn[s]] == pytwin.limbs(A)
        want32, _ = pytwin.round_int_f32(A, f)
        assert int(b32[s]) == want32
    # binary32 and 16-bit inputs, equal segments
    bits32 = synth.gen.bits("c2f32", 3, 64 * 37)
    b64, b32, fl, _ = oracle.sum_segments(bits32.view(np.float32), seg_len=37)
    for s in range(64):
        A, f = pytwin.exact_int_f32(bits32[s * 37:(s + 1) * 37])
        assert int(b64[s]) == pytwin.bits_of(pytwin.round_int(A, f)[0])
        assert int(b32[s]) == pytwin.round_int_f32(A, f)[0]
    for fmt in ("f16", "bf16"):
        bits16 = synth.gen.bits("c2" + fmt, 3, 50 * 41)
        b64, b32, fl, _ = oracle.sum_segments(bits16, seg_len=41, fmt=fmt)
        for s in range(50):
            A, f = pytwin.exact_int_h16(bits16[s * 41:(s + 1) * 41], fmt)
            assert int(b64[s]) == pytwin.bits_of(pytwin.round_int(A, f)[0]), (fmt, s)
