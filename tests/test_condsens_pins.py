"""Pins of the condition-number-sensitive oracle (oracle/condsens.py), CPU only.

Each pin checks the oracle against something other than itself: exact rational sums
(fractions.Fraction of a binary64 is exact), the standard library's correctly rounded
conversion and math.nextafter for the faithful bracket, hand-derived digits, and the
invariants Lemma 1 and the truncation definition fix (value preservation, digit range,
active-index rule, dropped magnitude). A plausible slip - a wrong carry sign or index, a
dropped carry entry, truncating the wrong end, a wrong eps_min - fails one of them."""
from __future__ import annotations

import math
import random
import struct
from fractions import Fraction

import pytest

from oracle import condsens as cs

R = 1 << 52
U = Fraction(1, 1 << 1074)


def exact(xs) -> Fraction:
    return sum((Fraction(x) for x in xs), Fraction(0))


def faithful(y: float, S: Fraction) -> bool:
    """y is one of the two floating-point neighbours of S (RD(S) or RU(S))."""
    if math.isinf(y):
        return False
    fy = Fraction(y)
    if fy == S:
        return True
    if fy < S:
        nxt = math.nextafter(y, math.inf)
        return math.isinf(nxt) or Fraction(nxt) > S
    prv = math.nextafter(y, -math.inf)
    return math.isinf(prv) or Fraction(prv) < S


def b2f(b: int) -> float:
    return struct.unpack("<d", struct.pack("<Q", b))[0]


def rand_double(rng, emin=1, emax=2046, subnormal=0.05) -> float:
    s = rng.getrandbits(1)
    if rng.random() < subnormal:
        e = 0
    else:
        e = rng.randint(emin, emax)
    return b2f((s << 63) | (e << 52) | rng.getrandbits(52))


def rand_sparse(rng, nnz=None) -> dict:
    """A random regularized sparse superaccumulator, boundary digits over-represented."""
    nnz = rng.randint(0, 12) if nnz is None else nnz
    idx = rng.sample(range(42), nnz)
    Y = {}
    for i in idx:
        c = rng.random()
        if c < 0.2:
            d = R - 1
        elif c < 0.4:
            d = R - 2
        elif c < 0.5:
            d = 1
        else:
            d = rng.randint(1, R - 1)
        Y[i] = d if rng.getrandbits(1) else -d
    if 41 in Y:                                  # keep |value| inside the window's range
        Y[41] = max(-(1 << 28), min(1 << 28, Y[41]))
    return Y


# ------------------------------------------------------------------------------------------
# leaves
# ------------------------------------------------------------------------------------------
def test_leaf_hand_derived():
    # 1.0: e = 1023 -> k = 1022 = 19*52 + 34, M = 2^52: M 2^34 = 2^86 = 2^34 R -> {20: 2^34}
    assert cs.leaf(1.0) == ({20: 1 << 34}, 0)
    # -1.5: M = 3 * 2^51, v = 3 * 2^85 = 3 * 2^33 R -> {20: -3 * 2^33}
    assert cs.leaf(-1.5) == ({20: -3 << 33}, 0)
    # least subnormal: e = 0, m = 1 -> k = 0, {0: 1}
    assert cs.leaf(b2f(1)) == ({0: 1}, 0)
    # DBL_MAX: k = 2045 = 39*52 + 17, M = 2^53 - 1: (2^53-1) 2^17 = (2^70 - 2^17) -> lo, hi
    v = ((1 << 53) - 1) << 17
    assert cs.leaf(b2f(0x7FEFFFFFFFFFFFFF)) == ({39: v % R, 40: v >> 52}, 0)
    assert cs.leaf(0.0) == ({}, 0) and cs.leaf(-0.0) == ({}, 0)
    assert cs.leaf(math.inf) == ({}, cs.F_PINF) and cs.leaf(-math.inf) == ({}, cs.F_NINF)
    assert cs.leaf(math.nan)[1] == cs.F_NAN


def test_leaf_value_and_range():
    rng = random.Random(1)
    for _ in range(20000):
        x = rand_double(rng)
        Y, f = cs.leaf(x)
        assert f == 0 and len(Y) <= 2
        assert cs.value(Y) == Fraction(x)
        assert all(0 < abs(d) <= R - 1 for d in Y.values())
        if len(Y) == 2:
            i, j = sorted(Y)
            assert j == i + 1


# ------------------------------------------------------------------------------------------
# Lemma 1 sums of sparse superaccumulators
# ------------------------------------------------------------------------------------------
def test_lemma1_sum_value_range_and_active_indices():
    rng = random.Random(2)
    for _ in range(20000):
        Y, Z = rand_sparse(rng), rand_sparse(rng)
        S = cs.lemma1_sum(Y, Z)
        assert cs.value(S) == cs.value(Y) + cs.value(Z)                 # exact
        assert all(0 < abs(d) <= R - 1 for d in S.values())              # regularized, no zeros
        allowed = set(Y) | set(Z) | {i + 1 for i in set(Y) | set(Z)}
        assert set(S) <= allowed                                         # carries move one digit


def test_lemma1_boundary_cases_by_hand():
    # P = R-1 carries (C = +1): (R-1) + 0 -> S_i = -1, S_{i+1} = +1  (Lemma 1, Case 1)
    assert cs.lemma1_sum({5: R - 1}, {}) == {5: -1, 6: 1}
    # P = -(R-1) -> C = -1: S_i = +1, S_{i+1} = -1 (Case 2)
    assert cs.lemma1_sum({5: -(R - 1)}, {}) == {5: 1, 6: -1}
    # P = R-2: no carry
    assert cs.lemma1_sum({5: R - 2}, {}) == {5: R - 2}
    # 2(R-1) = 2R-2 -> W = R-2, carry 1; incoming carry from below: (R-1)+(R-1) at 4 and 5
    assert cs.lemma1_sum({4: R - 1, 5: R - 1}, {4: R - 1, 5: R - 1}) == {4: R - 2, 5: R - 1, 6: 1}
    # cancellation leaves the index inactive
    assert cs.lemma1_sum({7: 12345}, {7: -12345}) == {}


# ------------------------------------------------------------------------------------------
# truncation
# ------------------------------------------------------------------------------------------
def test_truncate_keeps_most_significant_and_bounds_dropped():
    rng = random.Random(3)
    for _ in range(5000):
        Y = rand_sparse(rng)
        r = rng.choice([1, 2, 3, 4, 16])
        T, cut = cs.truncate(Y, r)
        assert len(T) == min(r, len(Y))
        assert set(T) == set(sorted(Y, reverse=True)[:r])
        assert all(T[i] == Y[i] for i in T)
        if cut is None:
            assert T == Y
        else:
            assert cut == min(T) and all(i < cut for i in set(Y) - set(T))
            assert abs(cs.value(Y) - cs.value(T)) < R ** cut * U       # < R^cut units


# ------------------------------------------------------------------------------------------
# the tree and the iteration
# ------------------------------------------------------------------------------------------
def test_tree_without_truncation_is_exact():
    rng = random.Random(4)
    for n in list(range(1, 40)) + [100, 257, 1000]:
        xs = [rand_double(rng) for _ in range(n)]
        t = cs.tree_sum([cs.leaf(x)[0] for x in xs], 256)
        assert t.e_cut is None and t.ntrunc == 0
        assert cs.value(t.root) == exact(xs)


def test_tree_shape_complete_binary_over_index_order():
    """Reading C2: n = 3 is ((x0, x1), x2) - the right child of the root's left... the last
    leaf passes up unchanged. With r = 1 the shape decides what survives:
    ((2^60, 1), 2^-60) keeps 2^60 after the first sum (1 is cut), then adds 2^-60 and cuts it."""
    xs = [2.0 ** 60, 1.0, 2.0 ** -60]
    t = cs.tree_sum([cs.leaf(x)[0] for x in xs], 1)
    assert cs.value(t.root) == Fraction(2 ** 60)
    assert t.ntrunc == 2
    # the other shape (x0, (x1, x2)) would keep the digit of 1 + 2^-60 first; a balanced tree over
    # 4 leaves pairs (x0, x1) and (x2, x3)
    xs4 = [1.0, 2.0 ** -200, 2.0 ** 200, -(2.0 ** 200)]
    t4 = cs.tree_sum([cs.leaf(x)[0] for x in xs4], 1)
    assert cs.value(t4.root) == Fraction(1)                 # (1 + tiny -> 1) + (big - big = 0)


def _cases():
    rng = random.Random(5)
    out = []
    for n in (1, 2, 3, 5, 8, 17, 64, 333, 1000):
        out.append(("wide", [rand_double(rng) for _ in range(n)]))
        out.append(("positive", [abs(rand_double(rng, 900, 1100, 0)) for _ in range(n)]))
        out.append(("narrow", [rand_double(rng, 1013, 1033, 0) for _ in range(n)]))
    for n in (4, 16, 200, 2000):                               # c3-like: (a, -a) pairs + tiny residue
        a = [rand_double(rng, 1023, 1623, 0) for _ in range(n)]
        t = [rand_double(rng, 123, 223, 0) for _ in range(max(1, n // 50))]
        xs = a + [-v for v in a] + t
        rng.shuffle(xs)
        out.append(("cancel", xs))
    out.append(("zero", [1.0, -1.0, 2.0 ** 900, -(2.0 ** 900)]))
    out.append(("subnormal", [b2f(rng.getrandbits(52)) for _ in range(300)]))
    out.append(("overflow", [b2f(0x7FEFFFFFFFFFFFFF)] * 3))
    out.append(("edge", [b2f(0x7FEFFFFFFFFFFFFF), b2f(0x7C9FFFFFFFFFFFFF)]))   # DBL_MAX + 2^969 - ...
    return out


@pytest.mark.parametrize("rule", [1, 2])
def test_condsens_result_is_faithful(rule):
    for kind, xs in _cases():
        S = exact(xs)
        res = cs.condsens_sum(xs, rule=rule)
        if res.exact:
            # no truncation anywhere: y is the RN-even rounding of the exact sum
            try:
                want = float(S)
            except OverflowError:
                want = math.inf if S > 0 else -math.inf
            assert res.value == want or (math.isnan(want) and math.isnan(res.value)), kind
        else:
            assert faithful(res.value, S), (kind, res.value, float(S))
            # the reading-C3 bound the stopping condition relies on: |S - T| < n eps_min
            T = cs.value(res.root)
            assert abs(S - T) < len(xs) * R ** res.e_cut * U, kind
        assert res.r in (2, 4, 16, 256) and res.iterations == {2: 1, 4: 2, 16: 3, 256: 4}[res.r]


def test_well_conditioned_inputs_stop_early():
    """C(X) = 1 (all terms of one sign): every partial sum is at most the total, so each node's
    cut is >= r-1 digits below the root's top digit; with r = 4 that leaves >= 2*52 bits of margin,
    so the iteration stops by r = 4 (the linear-work case of PAPER.md:1015-1022). With r = 2 it
    stops when the root's top digit carries enough bits - most random sets (radix 2^52)."""
    rng = random.Random(6)
    for n in (10, 100, 1000, 3000):
        xs = [abs(rand_double(rng, 1, 2030, 0.01)) for _ in range(n)]
        res = cs.condsens_sum(xs)
        assert res.iterations <= 2 and not res.exact and faithful(res.value, exact(xs))
    first = 0
    for _ in range(200):
        xs = [abs(rand_double(rng, 1, 2030, 0.01)) for _ in range(50)]
        res = cs.condsens_sum(xs)
        assert res.iterations <= 2
        first += res.iterations == 1
    assert first >= 120


def test_ill_conditioned_needs_more_iterations():
    rng = random.Random(7)
    a = [rand_double(rng, 1023, 1623, 0) for _ in range(500)]
    tiny = [rand_double(rng, 123, 223, 0) for _ in range(10)]
    xs = a + [-v for v in a] + tiny
    rng.shuffle(xs)
    res = cs.condsens_sum(xs)
    assert res.iterations >= 2 and faithful(res.value, exact(xs))


def test_literal_eps_min_is_not_sufficient():
    """Reading C3: with the paper's eps_min from the ROOT's least significant kept entry, this
    input stops at r = 2 with a y that is not a faithful rounding; with eps_min from the
    largest truncation index over all nodes it does not stop there.
    Leaves (8, complete tree): x0 = A (digits 7, 6), x1 = 2^-1074 R^5 (digit 5, cut at the
    first sum), x2 = -A, x4 = B (digits 3, 2), zeros elsewhere: (x0 + x1) -> A, (+ x2) -> 0,
    the root is B, but S = B + R^5 2^-1074."""
    A = b2f((((6 * 52 + 30) + 1) << 52) | 12345)           # k = 6*52 + 30: digits 6 and 7
    x1 = Fraction(R ** 5) * U
    B = b2f((((2 * 52 + 40) + 1) << 52) | 987654321)       # k = 2*52 + 40: digits 2 and 3
    xs = [A, float(x1), -A, 0.0, B, 0.0, 0.0, 0.0]
    assert Fraction(float(x1)) == x1
    n = len(xs)
    t = cs.tree_sum([cs.leaf(x)[0] for x in xs], 2)
    y = cs.rn(cs.value(t.root))
    S = exact(xs)
    assert t.root == cs.leaf(B)[0] and t.e_cut == 6            # the cut happened at index 6 (A's digits)
    i_r = min(t.root)                                          # the paper's E_{i_r}: index 2
    d = n * Fraction(R ** i_r) * U
    literal = cs.rn(Fraction(y) + d) == y and cs.rn(Fraction(y) - d) == y
    assert literal and not faithful(y, S)                      # the literal rule would stop wrongly
    assert not cs.stop_rule_1(y, n, t.e_cut)
    res = cs.condsens_sum(xs)
    assert res.iterations > 1 and faithful(res.value, S)


def test_rule2_implies_rule1():
    rng = random.Random(8)
    hits = 0
    for _ in range(3000):
        y = rand_double(rng, 1, 2046, 0.02)
        if y == 0:
            continue
        n = rng.choice([1, 2, 3, 7, 8, 1000, 1 << 20])
        e_cut = rng.randint(0, 41)
        if cs.stop_rule_2(y, n, e_cut):
            hits += 1
            assert cs.stop_rule_1(y, n, e_cut)
    assert hits > 100


def test_rule1_closed_form_edges():
    """(+) is exact RN-even: n eps_min exactly half an ulp above an even y does not move it,
    above an odd y it does; just below half an ulp never moves y."""
    # y = 1.0 (even mantissa): ulp = 2^-52; eps_min = 2^(52 E - 1074); E = 19 -> 2^-86
    y = 1.0
    E = 19
    eps = Fraction(R ** E) * U
    assert eps == Fraction(1, 1 << 86)
    n_half = 1 << 33                                           # n eps = 2^-53 = ulp/2 above y
    # below y the gap is 2^-53 (power of two): half of it is 2^-54, so n = 2^33 fails below
    assert not cs.stop_rule_1(y, n_half, E)
    assert cs.stop_rule_1(y, 1 << 32, E)                       # 2^-54: a tie below, y even -> stays
    assert not cs.stop_rule_1(y, (1 << 32) + 1, E)
    y_odd = 1.0 + 2.0 ** -52
    # gaps of 2^-52 on both sides: half of one is n = 2^33; a tie from an odd y moves it
    assert cs.stop_rule_1(y_odd, (1 << 33) - 1, E) and not cs.stop_rule_1(y_odd, 1 << 33, E)


def test_specials_and_zero():
    r = cs.condsens_sum([1.0, math.nan, 2.0])
    assert math.isnan(r.value) and r.flags & cs.F_NAN
    r = cs.condsens_sum([1.0, math.inf, -math.inf])
    assert math.isnan(r.value)
    r = cs.condsens_sum([1.0, -math.inf])
    assert r.value == -math.inf
    r = cs.condsens_sum([-0.0, -0.0])
    assert r.value == 0.0 and math.copysign(1, r.value) == 1 and r.exact
    r = cs.condsens_sum([])
    assert r.value == 0.0 and r.exact
