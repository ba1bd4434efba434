"""Index arithmetic at the sizes where 32-bit offsets would wrap (every kernel family once):
more than 2^32 ELEMENTS of 16-bit / 32-bit input (element indices), and more than 2^32 BYTES
(4 GiB) of binary64 input in the short-segment, CSR and strided paths (byte offsets). Each device
result is compared bit for bit with the oracle (oracle/) on the same bytes: values, flags and,
for the whole-array sums, the 34-limb canonical image. Inputs are seeded uniform finite bit
patterns (NaN/Inf patterns moved to finite ones), drawn on the device and copied to the host."""
from __future__ import annotations

import numpy as np
import pytest

import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def xs():
    import torch  # noqa: F401
    import paper_1605_05436_b200 as xsum
    xsum.build()
    return xsum


def finite_bits(n: int, fmt: str, seed: int):
    """n uniform finite bit patterns of fmt on the device (int tensor of the format's width)."""
    import torch
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    if fmt == "f64":
        x = torch.randint(-2 ** 63, 2 ** 63 - 1, (n,), dtype=torch.int64, device="cuda", generator=g)
        em = 0x7FF0000000000000
        return torch.where((x & em) == em, x ^ (1 << 52), x)
    if fmt == "f32":
        x = torch.randint(-2 ** 31, 2 ** 31 - 1, (n,), dtype=torch.int32, device="cuda", generator=g)
        return torch.where((x & 0x7F800000) == 0x7F800000, x ^ 0x800000, x)
    x = torch.randint(-32768, 32767, (n,), dtype=torch.int16, device="cuda", generator=g)
    em = 0x7C00 if fmt == "f16" else 0x7F80
    return torch.where((x & em) == em, x ^ 0x400, x)


def view(bits, fmt: str):
    import torch
    return bits.view({"f64": torch.float64, "f32": torch.float32, "f16": torch.float16,
                      "bf16": torch.bfloat16}[fmt])


def host(bits):
    return bits.cpu().numpy()


def test_f16_sum_beyond_2p32_elements(xs):
    n = (1 << 32) + (1 << 16) + 5
    b = finite_bits(n, "f16", 1)
    res, canon = xs.Accumulator().sum(view(b, "f16"), canon=True)
    got = xs.Result.from_bytes(res.cpu().numpy().tobytes())
    canon = canon.cpu().numpy().view(np.uint64)
    h = host(b).view(np.uint16)
    del b
    r, limbs = oracle.exact_sum(h, fmt="f16")
    assert got.count == n and got.bits == r.bits and got.flags == r.flags and (canon == limbs).all()


def test_f32_sum_beyond_2p32_elements(xs):
    n = (1 << 32) + 7
    b = finite_bits(n, "f32", 2)
    res, canon = xs.Accumulator().sum(view(b, "f32"), canon=True)
    got = xs.Result.from_bytes(res.cpu().numpy().tobytes())
    canon = canon.cpu().numpy().view(np.uint64)
    h = host(b).view(np.float32)
    del b
    r, limbs = oracle.exact_sum(h)
    assert got.count == n and got.bits == r.bits and got.flags == r.flags and (canon == limbs).all()


@pytest.mark.parametrize("fmt,seg_len,nseg", [("bf16", 4096, (1 << 20) + 2),     # K9q, > 2^32 elements
                                              ("bf16", 8, (1 << 29) + 3),        # K11 lanes, > 2^32 elements
                                              ("f64", 16, (1 << 25) + 7)])       # K11s, > 4 GiB
def test_equal_segments_beyond_32bit_offsets(xs, fmt, seg_len, nseg):
    b = finite_bits(seg_len * nseg, fmt, 3 + seg_len)
    vals, _, flags = xs.sum_segments(view(b, fmt), seg_len, flags=True)
    vals = vals.cpu().numpy()
    flags = flags.cpu().numpy().astype(np.uint32)
    h = host(b)
    del b
    if fmt == "f64":
        b64, _, fl, _ = oracle.sum_segments(h.view(np.float64), seg_len=seg_len)
        assert (vals.view(np.uint64) == b64).all()
    else:
        _, b32, fl, _ = oracle.sum_segments(h.view(np.uint16), seg_len=seg_len, fmt=fmt)
        assert (vals.view(np.uint32) == b32).all()
    assert (flags == fl).all()


def test_csr_segments_beyond_4gib(xs):
    """Ragged binary64 segments whose offsets pass 2^29 elements (4 GiB): a few long ones around
    the boundary, empty ones, and short ones after it."""
    import torch
    n = (1 << 29) + 4099
    b = finite_bits(n, "f64", 5)
    cuts = [0, 1, (1 << 28) + 3, (1 << 29) - 5, (1 << 29) - 5, (1 << 29) + 1, (1 << 29) + 17, (1 << 29) + 17,
            (1 << 29) + 2000, n]
    off = np.array(cuts, dtype=np.int64)
    vals, canon, flags = xs.sum_segments_csr(view(b, "f64"), torch.from_numpy(off).cuda(), canon=True, flags=True)
    h = host(b).view(np.float64)
    del b
    b64, _, fl, cn = oracle.sum_segments(h, offsets=off.astype(np.uint64), canon=True)
    assert (vals.cpu().numpy().view(np.uint64) == b64).all()
    assert (flags.cpu().numpy().astype(np.uint32) == fl).all()
    assert (canon.cpu().numpy().view(np.uint64) == cn).all()


def test_strided_f16_beyond_2p32_elements(xs):
    """exact_sum_dim over dim 0 of a [2^16 + 1, 2^16] binary16 matrix (K10h); 512 sampled
    columns (every 128th, plus the last) against the oracle's per-fibre sums."""
    rows, cols = (1 << 16) + 1, 1 << 16
    b = finite_bits(rows * cols, "f16", 6)
    out = xs.exact_sum_dim(view(b, "f16").view(rows, cols), 0)
    assert tuple(out.shape) == (cols,)
    got = out.cpu().numpy().view(np.uint32)
    pick = np.r_[np.arange(0, cols, 128), cols - 1]
    fib = host(b.view(rows, cols)[:, torch_index(pick)]).view(np.uint16)
    del b
    _, b32, _, _ = oracle.sum_segments(np.ascontiguousarray(fib.T).reshape(-1), seg_len=rows, fmt="f16")
    assert (got[pick] == b32).all()


def torch_index(a):
    import torch
    return torch.from_numpy(np.asarray(a, dtype=np.int64)).cuda()
