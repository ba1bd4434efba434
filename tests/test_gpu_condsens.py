"""GPU parity of the condition-number-sensitive sum (K12, xsum_sum_condsens; SURVEY.md §8(f) f4;
PAPER.md:851-965) against oracle/condsens.py (O3) and, at full size, against the exact oracle.

At oracle-sized inputs (spanning several chunks and passes of every r, with ragged tails) the
GPU must match O3 exactly: the last iteration's r, the iteration count, E_cut, the exact flag,
the root's sparse superaccumulator digit for digit (truncated iterations), the value bits and
flags, and the canonical image of the truncated root. At BASELINE sizes the result must be a
faithful rounding of the exact sum (O1 limbs), the truncation bound |S - T| < n eps_min must hold
(T from the returned canonical image), and the well-conditioned config must stop early."""
from __future__ import annotations

import math
import random
import struct
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from oracle import condsens as cs

pytestmark = pytest.mark.gpu

R = 1 << 52


@pytest.fixture(scope="module")
def xs():
    import torch  # noqa: F401
    import paper_1605_05436_b200 as xsum
    xsum.build()
    synth.build()
    return xsum


def b2f(b: int) -> float:
    return struct.unpack("<d", struct.pack("<Q", b))[0]


def f2b(x: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def rand_double(rng, emin=1, emax=2046, subnormal=0.05) -> float:
    s = rng.getrandbits(1)
    e = 0 if rng.random() < subnormal else rng.randint(emin, emax)
    return b2f((s << 63) | (e << 52) | rng.getrandbits(52))


def to_dev(xs_list, offset: int = 0):
    import torch
    a = np.array(xs_list, dtype=np.float64)
    buf = torch.zeros(a.size + 2, dtype=torch.float64, device="cuda")
    t = buf[offset:offset + a.size]
    t.copy_(torch.from_numpy(a))
    return t


def faithful(y: float, S: Fraction) -> bool:
    if math.isinf(y) or math.isnan(y):
        return False
    fy = Fraction(y)
    if fy == S:
        return True
    if fy < S:
        nxt = math.nextafter(y, math.inf)
        return math.isinf(nxt) or Fraction(nxt) > S
    prv = math.nextafter(y, -math.inf)
    return math.isinf(prv) or Fraction(prv) < S


def compare(xsum, vals, rule=1, offset=0, what=""):
    d = to_dev(vals, offset)
    res, info, canon = xsum.condsens_sum(d, rule)
    o = cs.condsens_sum(vals, rule=rule)
    assert info.r == o.r and info.iterations == o.iterations and info.exact == o.exact, \
        (what, info, (o.r, o.iterations, o.exact))
    assert info.rule == rule
    if o.r <= 16:                          # the truncated tree: identical root digits and E_cut
        assert info.e_cut == o.e_cut, (what, info.e_cut, o.e_cut)
        assert info.root == o.root, (what, info.root, o.root)
        T = cs.value(o.root)
    else:                                  # the exact pass: the exact sum itself
        assert info.e_cut is None and info.root == {}
        T = sum((Fraction(v) for v in vals if math.isfinite(v)), Fraction(0))
    if math.isnan(o.value):
        assert math.isnan(res.value), what
    else:
        assert res.bits == f2b(o.value), (what, res.value, o.value)
    assert res.flags & 7 == o.flags & 7 or (o.flags & 7 == 0 and res.flags & 7 == 0), what
    assert res.count == len(vals)
    A = T * (1 << 1074)
    assert A.denominator == 1
    assert (canon == oracle.int_to_limbs(int(A))).all(), what
    return res, info, o


def _families(rng, n):
    yield "wide", [rand_double(rng) for _ in range(n)]
    yield "positive", [abs(rand_double(rng, 1, 2030, 0.01)) for _ in range(n)]
    yield "narrow", [rand_double(rng, 1013, 1033, 0) for _ in range(n)]
    a = [rand_double(rng, 1023, 1623, 0) for _ in range(n // 2)]
    t = [rand_double(rng, 123, 223, 0) for _ in range(max(1, n // 64))]
    c = a + [-v for v in a] + t
    rng.shuffle(c)
    yield "cancel", c[:n] if len(c) >= n else c


@pytest.mark.parametrize("n", [1, 2, 3, 31, 32, 33, 255, 256, 257, 1023, 1025, 4095, 4096, 4097, 9000,
                               16383, 16384, 16385])
def test_condsens_matches_oracle_sizes(xs, n):
    rng = random.Random(1000 + n)
    for kind, vals in _families(rng, n):
        compare(xs, vals, 1, what=f"{kind} n={n}")


@pytest.mark.parametrize("rule", [1, 2])
def test_condsens_multi_pass(xs, rule):
    """Sizes past one chunk of every r (r = 2: 16384 leaves, r = 4: 4096, r = 16: 1024 per warp)
    and so through a second pass of every r, misaligned base."""
    rng = random.Random(7 + rule)
    for kind, vals in _families(rng, 70_001):
        if kind in ("wide", "cancel"):
            compare(xs, vals, rule, offset=1, what=f"{kind} 70001 rule {rule}")


def test_condsens_exact_and_special_paths(xs):
    rng = random.Random(11)
    # nothing truncated (few distinct digits): exact at r = 2
    compare(xs, [1.0] * 1000, what="ones")
    compare(xs, [0.0, -0.0] * 50, what="zeros")
    compare(xs, [], what="empty")
    # the reading-C3 counterexample: must not stop at r = 2
    A = b2f((((6 * 52 + 30) + 1) << 52) | 12345)
    x1 = float(Fraction(R ** 5, 1 << 1074))
    B = b2f((((2 * 52 + 40) + 1) << 52) | 987654321)
    _, info, o = compare(xs, [A, x1, -A, 0.0, B, 0.0, 0.0, 0.0], what="counterexample")
    assert info.iterations > 1
    # specials
    v = [rand_double(rng) for _ in range(5000)]
    for sp in (math.nan, math.inf, -math.inf):
        w = list(v)
        w[1234] = sp
        compare(xs, w, what=f"special {sp}")
    w = list(v)
    w[10], w[4000] = math.inf, -math.inf
    compare(xs, w, what="inf-inf")
    # overflow of the root value: the iteration runs to the exact pass (y = +-inf is never accepted)
    compare(xs, [b2f(0x7FEFFFFFFFFFFFFF)] * 7, what="overflow")
    # sums that need every iteration: cancelling pairs with a tiny residue
    a = [rand_double(rng, 1023, 2000, 0) for _ in range(3000)]
    c = a + [-u for u in a] + [rand_double(rng, 1, 60, 0) for _ in range(3)]
    rng.shuffle(c)
    _, info, _ = compare(xs, c, what="deep cancel")
    assert info.iterations >= 3


@pytest.mark.parametrize("rule", [1, 2])
def test_condsens_random_fuzz(xs, rule):
    rng = random.Random(99 + rule)
    for trial in range(60):
        n = rng.choice([5, 17, 100, 513, 2000, 5000])
        fam = list(_families(rng, n))
        kind, vals = fam[trial % len(fam)]
        compare(xs, vals, rule, offset=trial & 1, what=f"fuzz {trial} {kind} {n}")


@pytest.mark.parametrize("cfg", ["c2", "c3"])
def test_condsens_full_config_faithful(xs, cfg):
    """BASELINE sizes (c2: 2^28; c3: 2^28 + 2^20, ill-conditioned): y is a faithful rounding of
    the exact sum (O1), the truncated root T (canonical image) obeys |S - T| < n eps_min, and
    the well-conditioned c2 stops within two iterations while c3 needs the deeper ones."""
    import torch
    d = synth.device_generate(cfg)
    n = d.numel()
    res, info, canon = xs.condsens_sum(d, 1)
    del d
    torch.cuda.empty_cache()
    r_ex, limbs = oracle.exact_sum(synth.host_generate(cfg))       # c3: pre-permutation order
    S = Fraction(oracle.limbs_to_int(limbs), 1 << 1074)
    T = Fraction(oracle.limbs_to_int(canon), 1 << 1074)
    if info.exact:
        assert res.bits == r_ex.bits
    else:
        assert faithful(res.value, S), (cfg, res.value, float(S))
        assert abs(S - T) < n * Fraction(R ** info.e_cut, 1 << 1074)
    if cfg == "c2":
        assert info.iterations <= 2 and not info.exact
    else:
        assert info.iterations >= 2



def test_condsens_buffer_checks(xs):
    """Caller-provided buffers: a work buffer that is not a 256-B aligned uint8 CUDA tensor is
    refused before the call; a reused buffer gives the same result as a fresh one."""
    import torch
    d = to_dev([1.0, 2.0 ** -60, -3.5] * 1000)
    nb = xs.condsens_work_bytes(d.numel())
    for bad in (torch.empty(nb, dtype=torch.float32, device="cuda"),
                torch.empty(nb + 1, dtype=torch.uint8, device="cuda")[1:],
                torch.empty(nb, dtype=torch.uint8)):
        with pytest.raises(TypeError):
            xs.sum_condsens(d, 1, work=bad)
    work = torch.empty(nb, dtype=torch.uint8, device="cuda")
    r1, i1, _ = xs.sum_condsens(d, 1, work=work)
    r2, i2, _ = xs.sum_condsens(d, 1)
    assert bytes(r1.cpu().numpy()) == bytes(r2.cpu().numpy()) and bytes(i1.cpu().numpy()) == bytes(i2.cpu().numpy())
