"""GPU parity for 16-bit inputs (binary16 / bfloat16): the CUDA path through
the C-ABI vs the oracle, bit for bit (rounded binary64 and binary32, direction, flags and the
canonical image). Inputs are seeded bit patterns; expected values come only from oracle/."""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

GOLDEN_H16 = os.path.join(os.path.dirname(__file__), "golden", "rounding_edges_h16.txt")
EMASK = {"f16": 0x7C00, "bf16": 0x7F80}


@pytest.fixture(scope="module")
def xs():
    import torch  # noqa: F401
    import paper_1605_05436_b200 as xsum
    xsum.build()
    return xsum


def patterns(n: int, seed: int, fmt: str, specials: bool = False, narrow: tuple | None = None) -> np.ndarray:
    """Seeded uint16 bit patterns: uniform over all finite patterns (every exponent, subnormals,
    zeros, both signs), or exponent fields in `narrow` = (lo, hi); optional NaN/Inf patterns."""
    rng = np.random.default_rng(seed)
    b = rng.integers(0, 1 << 16, size=n, dtype=np.uint32).astype(np.uint16)
    t = 10 if fmt == "f16" else 7
    if narrow is not None:
        e = rng.integers(narrow[0], narrow[1] + 1, size=n, dtype=np.uint32).astype(np.uint16)
        b = (b & np.uint16(0x8000 | ((1 << t) - 1))) | (e << np.uint16(t)).astype(np.uint16)
    em = EMASK[fmt]
    fin = (b & em) == em
    b[fin] ^= np.uint16(1 << t)                   # move NaN/Inf patterns to the largest finite exponent
    if specials and n:
        idx = rng.choice(n, size=min(n, 9), replace=False)
        b[idx] = rng.choice(np.array([em, 0x8000 | em, em | 1, em | 0x8000 | 3], dtype=np.uint16), size=idx.size)
    return b


def to_dev16(b: np.ndarray, fmt: str, offset: int = 0):
    import torch
    dt = torch.float16 if fmt == "f16" else torch.bfloat16
    buf = torch.empty(b.size + 8, dtype=torch.int16, device="cuda")
    assert buf.data_ptr() % 16 == 0
    t = buf[offset:offset + b.size]
    t.copy_(torch.from_numpy(np.ascontiguousarray(b).view(np.int16)))
    return t.view(dt)


def check(xs, res, canon, ref, what):
    r, limbs = ref
    assert res.bits == r.bits, f"{what}: value {res.bits:016x} != oracle {r.bits:016x}"
    assert res.bits_f32 == r.bits_f32, f"{what}: binary32 {res.bits_f32:08x} != {r.bits_f32:08x}"
    assert res.direction == r.direction and res.flags == r.flags, f"{what}: {res} vs {r}"
    assert res.sig53 == r.sig53 and res.exp2 == r.exp2 and res.count == r.count, what
    if canon is not None:
        assert (np.asarray(canon, dtype=np.uint64) == limbs).all(), f"{what}: canonical image differs"


@pytest.mark.parametrize("fmt", ["f16", "bf16"])
def test_golden_h16(xs, fmt):
    for line in open(GOLDEN_H16):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        name, f, ins, o64, o32, _ = [p.strip() for p in line.split("|")]
        if f != fmt:
            continue
        b = np.array([int(h, 16) for h in ins.split(",")], dtype=np.uint16)
        res, canon = xs.exact_sum(to_dev16(b, fmt))
        assert res.bits == int(o64, 16) and res.bits_f32 == int(o32, 16), name
        check(xs, res, canon, oracle.exact_sum(b, fmt=fmt), name)


@pytest.mark.parametrize("fmt", ["f16", "bf16"])
@pytest.mark.parametrize("n", [0, 1, 2, 7, 8, 9, 63, 4095, 4096, 16384 + 5, 65536 + 3, 148 * 16384 + 13, 3_000_001])
@pytest.mark.parametrize("off", [0, 1, 7])
def test_h16_sizes_alignment(xs, fmt, n, off):
    b = patterns(n, n * 3 + off, fmt)
    ref = oracle.exact_sum(b, fmt=fmt)
    d = to_dev16(b, fmt, off)
    res, canon = xs.exact_sum(d)
    check(xs, res, canon, ref, f"{fmt} fused n={n} off={off}")
    acc = xs.Accumulator().add(d)
    res2, canon2 = acc.exact()
    check(xs, res2, canon2, ref, f"{fmt} acc n={n} off={off}")


@pytest.mark.parametrize("fmt", ["f16", "bf16"])
@pytest.mark.parametrize("blocks", [1, 3])
def test_h16_bin_windows_and_specials(xs, fmt, blocks):
    # many bin windows per lane (the bfloat16 window is 511 summands), worst-case bins: every
    # summand the largest finite magnitude of one exponent group, all of one sign
    n = 40 * 16384 * blocks + 333
    b = patterns(n, blocks, fmt)
    acc = xs.Accumulator().set_grid_limit(blocks)
    res, canon = acc.sum(to_dev16(b, fmt), canon=True)
    check(xs, xs.Result.from_bytes(res.cpu().numpy().tobytes()), canon.cpu().numpy().view(np.uint64),
          oracle.exact_sum(b, fmt=fmt), f"{fmt} windows blocks={blocks}")
    top = np.uint16(0x7BFF if fmt == "f16" else 0x7F7F)
    w = np.full(n, top, dtype=np.uint16)
    res, canon = acc.reset().add(to_dev16(w, fmt, 3)).exact()
    check(xs, res, canon, oracle.exact_sum(w, fmt=fmt), f"{fmt} worst-case bins")
    y = patterns(n, blocks + 10, fmt, specials=True)
    res, canon = acc.reset().add(to_dev16(y, fmt, 1)).exact()
    check(xs, res, canon, oracle.exact_sum(y, fmt=fmt), f"{fmt} specials blocks={blocks}")


@pytest.mark.parametrize("fmt", ["f16", "bf16"])
def test_h16_narrow_exponents_and_cancellation(xs, fmt):
    # a narrow exponent range (all summands in one or two bin groups: the bins' hot spot),
    # then x followed by -x: the exact sum is +0.0 (R9)
    lo, hi = (14, 16) if fmt == "f16" else (126, 128)
    b = patterns(5_000_000, 42, fmt, narrow=(lo, hi))
    d = to_dev16(b, fmt)
    res, canon = xs.exact_sum(d)
    check(xs, res, canon, oracle.exact_sum(b, fmt=fmt), f"{fmt} narrow")
    import torch
    both = torch.cat([d, -d])
    res, canon = xs.exact_sum(both)
    assert res.bits == 0 and not np.asarray(canon).any()


def test_h16_mixed_with_binary64_in_one_state(xs):
    import torch
    a = patterns(1_000_003, 5, "f16")
    c = patterns(777_777, 6, "bf16")
    x = np.random.default_rng(1).standard_normal(123_457) * 1e3
    acc = xs.Accumulator().add(to_dev16(a, "f16", 1)).add(torch.from_numpy(x).cuda()).add(to_dev16(c, "bf16"))
    res, canon = acc.exact()
    oa = oracle.Accumulator().add(a.view(np.float16)).add(x).add(c, fmt="bf16")
    check(xs, res, canon, (oa.result(), oa.limbs), "mixed f16 + f64 + bf16")


def test_h16_status_codes(xs):
    import torch
    L = xs.lib()
    acc = xs.Accumulator()
    h = torch.zeros(16, dtype=torch.float16, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    assert L.xsum_accumulate_f16(acc.handle, h.data_ptr() + 1, 3, st) == xs.EINVAL    # not 2-B aligned
    assert L.xsum_accumulate_bf16(acc.handle, None, 3, st) == xs.EINVAL
    assert L.xsum_accumulate_bf16(acc.handle, h.data_ptr(), 0, st) == xs.OK
    assert L.xsum_sum_f16(acc.handle, h.data_ptr(), 3, None, None, st) == xs.EINVAL
    assert L.xsum_accumulate_f16(acc.handle, h.data_ptr(), 2 ** 63, st) == xs.ECAPACITY


@pytest.mark.parametrize("fmt", ["f16", "bf16"])
def test_h16_signed_zeros_and_subnormals(xs, fmt):
    # -0 has M = 0 with the sign bit set (the case a sign-extension slip gets wrong), and
    # subnormals have no hidden bit (R2); alone, mixed, and as a block-sized run
    rng = np.random.default_rng(3)
    subs = rng.integers(1, 1 << (10 if fmt == "f16" else 7), size=5000, dtype=np.uint32).astype(np.uint16)
    subs |= (rng.integers(0, 2, size=5000, dtype=np.uint32) << 15).astype(np.uint16)
    for b in (np.array([0x8000], np.uint16), np.array([0x8000, 0x0000, 0x8000], np.uint16),
              np.full(40000, 0x8000, np.uint16), subs, np.concatenate([subs, np.full(777, 0x8000, np.uint16)])):
        res, canon = xs.exact_sum(to_dev16(b, fmt, 1))
        check(xs, res, canon, oracle.exact_sum(b, fmt=fmt), f"{fmt} zeros/subnormals n={b.size}")
