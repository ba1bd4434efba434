"""GPU parity of segmented exact sums for every input format (xsum_sum_segments_ex; SURVEY.md
§8(f) f1 x f2): per segment, the binary32 (and for binary64 inputs also the binary64) rounding,
the flags and the canonical image vs the oracle, for equal and CSR segments, ragged lengths,
misaligned bases, specials, subnormals, signed zeros and segments longer than a flush window."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

TORCH_DT = {"f32": "float32", "f16": "float16", "bf16": "bfloat16"}


@pytest.fixture(scope="module")
def xs():
    import torch  # noqa: F401
    import paper_1605_05436_b200 as xsum
    xsum.build()
    synth.build()
    return xsum


def bits_data(fmt: str, n: int, seed: int) -> np.ndarray:
    """Seeded bit patterns (uint32 for f32, uint16 otherwise): all exponents, subnormals, zeros,
    a few NaN / Inf."""
    rng = np.random.default_rng(seed)
    if fmt == "f32":
        b = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
        em, t = 0x7F800000, 23
        spec = np.array([0x7F800000, 0xFF800000, 0x7FC00001, 0x80000000, 0x00000001], dtype=np.uint32)
    else:
        b = rng.integers(0, 1 << 16, size=n, dtype=np.uint32).astype(np.uint16)
        em, t = (0x7C00, 10) if fmt == "f16" else (0x7F80, 7)
        spec = np.array([em, 0x8000 | em, em | 1, 0x8000, 0x0001], dtype=np.uint16)
    fin = (b & em) == em
    b[fin] ^= b.dtype.type(1 << t)
    if n > 50:
        idx = rng.choice(n, size=max(1, n // 5000), replace=False)
        b[idx] = rng.choice(spec, size=idx.size)
    return b


def to_dev(b: np.ndarray, fmt: str, offset: int):
    import torch
    dt = getattr(torch, TORCH_DT[fmt])
    it = torch.int32 if fmt == "f32" else torch.int16
    buf = torch.empty(b.size + 8, dtype=it, device="cuda")
    t = buf[offset:offset + b.size]
    t.copy_(torch.from_numpy(b.view(np.int32 if fmt == "f32" else np.int16)))
    return t.view(dt)


def ref_of(fmt: str, seg: np.ndarray):
    if fmt == "f32":
        return oracle.exact_sum(seg.view(np.float32))
    return oracle.exact_sum(seg, fmt=fmt)


def check_segments(xs, fmt, b, bounds, vals, canon, flags, what):
    v = vals.cpu().numpy().view(np.uint32)
    cn = canon.cpu().numpy().view(np.uint64)
    fl = flags.cpu().numpy().view(np.uint32)
    for s, (a, e) in enumerate(bounds):
        r, limbs = ref_of(fmt, b[a:e])
        assert v[s] == r.bits_f32, f"{what} seg {s}: {v[s]:08x} != {r.bits_f32:08x}"
        assert fl[s] == r.flags and (cn[s] == limbs).all(), f"{what} seg {s}"


@pytest.mark.parametrize("fmt", ["f32", "f16", "bf16"])
@pytest.mark.parametrize("seg_len,off", [(1, 0), (3, 1), (8, 0), (9, 3), (255, 1), (1000, 0), (4096, 2),
                                         (70_001, 1)])
def test_equal_segments(xs, fmt, seg_len, off):
    nseg = max(1, min(64, 300_000 // seg_len))
    b = bits_data(fmt, nseg * seg_len, seg_len + off)
    vals, canon, flags = xs.sum_segments(to_dev(b, fmt, off), seg_len, canon=True, flags=True)
    check_segments(xs, fmt, b, [(s * seg_len, (s + 1) * seg_len) for s in range(nseg)], vals, canon, flags,
                   f"{fmt} L={seg_len} off={off}")


@pytest.mark.parametrize("fmt", ["f32", "f16", "bf16"])
def test_csr_segments_ragged(xs, fmt):
    import torch
    rng = np.random.default_rng(9)
    lens = rng.integers(0, 3000, size=150)
    lens[::17] = 0
    lens[5] = 90_000                                     # longer than a lane's flush window
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    b = bits_data(fmt, int(offs[-1]), 77)
    vals, canon, flags = xs.sum_segments_csr(to_dev(b, fmt, 1), torch.from_numpy(offs).cuda(), canon=True,
                                             flags=True)
    check_segments(xs, fmt, b, list(zip(offs[:-1], offs[1:])), vals, canon, flags, f"{fmt} csr")


def test_binary64_segments_binary32_output(xs):
    """xsum_sum_segments_ex on binary64 input writes both roundings (each once from the exact sum)."""
    import ctypes

    import torch
    x = synth.gen.generate("c5", 0, 64 * 4096)
    d = torch.from_numpy(x).cuda()
    out = torch.empty(64, dtype=torch.float64, device="cuda")
    out32 = torch.empty(64, dtype=torch.float32, device="cuda")
    rc = xs.lib().xsum_sum_segments_ex(d.data_ptr(), 0, 64, 4096, None, out.data_ptr(), out32.data_ptr(), None,
                                       None, torch.cuda.current_stream().cuda_stream)
    assert rc == xs.OK
    o64, o32 = out.cpu().numpy().view(np.uint64), out32.cpu().numpy().view(np.uint32)
    for s in range(64):
        r, _ = oracle.exact_sum(x[s * 4096:(s + 1) * 4096])
        assert o64[s] == r.bits and o32[s] == r.bits_f32, s
    st = torch.cuda.current_stream().cuda_stream
    assert xs.lib().xsum_sum_segments_ex(d.data_ptr(), 7, 1, 1, None, out.data_ptr(), None, None, None, st) == \
        xs.EINVAL
    assert xs.lib().xsum_sum_segments_ex(d.data_ptr(), 0, 1, 1, None, None, None, None, None, st) == xs.EINVAL
    del ctypes


@pytest.mark.parametrize("fmt", ["f32", "bf16"])
def test_exact_sum_dim_formats(xs, fmt):
    b = bits_data(fmt, 37 * 1001, 5)
    t = to_dev(b, fmt, 0).reshape(37, 1001)
    for dim in (0, 1):
        out = xs.exact_sum_dim(t, dim).cpu().numpy().view(np.uint32)
        bb = b.reshape(37, 1001)
        fib = bb if dim == 1 else bb.T
        for i, row in enumerate(fib):
            r, _ = ref_of(fmt, np.ascontiguousarray(row))
            assert out[i] == r.bits_f32, (fmt, dim, i)


@pytest.mark.parametrize("fmt", ["f32", "f16", "bf16"])
def test_host_buffer_streaming_formats(xs, fmt):
    """xsum_accumulate_host_ex: pinned host tensors of each format through a 2 MiB staging buffer
    (several double-buffered chunks) vs the oracle."""
    import torch
    n = 3_000_003
    b = bits_data(fmt, n, 123)
    dt = getattr(torch, TORCH_DT[fmt])
    host = torch.from_numpy(b.view(np.int32 if fmt == "f32" else np.int16)).view(dt).pin_memory()
    acc = xs.Accumulator().add_host(host, stage_bytes=2 << 20)
    res, canon = acc.exact()
    r, limbs = ref_of(fmt, b)
    assert res.bits == r.bits and res.bits_f32 == r.bits_f32 and res.flags == r.flags
    assert (canon == limbs).all() and res.count == n


@pytest.mark.parametrize("fmt", ["f32", "f16", "bf16"])
def test_segments_full_of_specials(xs, fmt):
    """A long segment made mostly of NaN / Inf patterns (more than a bin window per lane): the
    rare path cancels every one exactly; a segment of +Inf and finite values gives +Inf, one of
    only finite values next to it is unaffected."""
    import torch
    n = 70_000
    b = bits_data(fmt, 3 * n, 31)
    em = {"f32": 0x7F800000, "f16": 0x7C00, "bf16": 0x7F80}[fmt]
    pinf = b.dtype.type(em)
    b[: n - 5] = pinf                                   # segment 0: +Inf almost everywhere
    b[n: n + n // 2] = b.dtype.type(em | 1)             # segment 1: half NaN
    vals, canon, flags = xs.sum_segments(to_dev(b, fmt, 1), n, canon=True, flags=True)
    check_segments(xs, fmt, b, [(0, n), (n, 2 * n), (2 * n, 3 * n)], vals, canon, flags, f"{fmt} specials")


@pytest.mark.parametrize("fmt", ["f32", "f16", "bf16"])
def test_every_exponent_each_format(xs, fmt):
    """Every finite exponent field of the format with a random fraction and both signs: alone
    (segments of length 1: the bin / group / column-window placement of every exponent) and all
    together through the fused kernel, vs the oracle."""
    rng = np.random.default_rng(7)
    t, l = {"f32": (23, 8), "f16": (10, 5), "bf16": (7, 8)}[fmt]
    ut = np.uint32 if fmt == "f32" else np.uint16
    e = np.repeat(np.arange((1 << l) - 1, dtype=np.uint64), 2)
    fr = rng.integers(0, 1 << t, size=e.size, dtype=np.uint64)
    sg = np.tile(np.array([0, 1], dtype=np.uint64), e.size // 2)
    b = ((sg << np.uint64(t + l)) | (e << np.uint64(t)) | fr).astype(ut)
    d = to_dev(b, fmt, 0)
    vals, canon, flags = xs.sum_segments(d, 1, canon=True, flags=True)
    check_segments(xs, fmt, b, [(i, i + 1) for i in range(b.size)], vals, canon, flags, f"{fmt} exponents")
    res, cn = xs.exact_sum(d)
    r, limbs = ref_of(fmt, b)
    assert res.bits == r.bits and res.bits_f32 == r.bits_f32 and (cn == limbs).all()


@pytest.mark.parametrize("fmt", ["f32", "f16", "bf16"])
@pytest.mark.parametrize("seg_len,nseg", [(264, 37), (512, 101), (4096, 203), (8200, 9), (70_000, 5)])
def test_h16_equal_segments_values_only(xs, fmt, seg_len, nseg):
    """binary32 / 16-bit equal segments without canonical images (the quarter-warp kernels when the
    base is 16-B aligned and the length a multiple of 4 / 8): binary32 values, binary64 values and flags of
    every segment vs the oracle's per-segment sums - segments longer than a bin window (bfloat16:
    511 adds per lane), a partial last group of four, specials, and the fallback for a
    misaligned base."""
    import torch
    b = bits_data(fmt, seg_len * nseg, 700 + seg_len)
    b64, b32, fl, _ = oracle.sum_segments(b.view(np.float32) if fmt == "f32" else b, seg_len=seg_len,
                                          fmt=None if fmt == "f32" else fmt)
    for off in (0, 1):
        d = to_dev(b, fmt, off)
        v32, _, f = xs.sum_segments(d, seg_len, flags=True)
        assert (v32.cpu().numpy().view(np.uint32) == b32).all(), (fmt, seg_len, off)
        assert (f.cpu().numpy().view(np.uint32) == fl).all(), (fmt, seg_len, off)
        out = torch.empty(nseg, dtype=torch.float64, device="cuda")
        rc = xs.lib().xsum_sum_segments_ex(d.data_ptr(), {"f32": 1, "f16": 2, "bf16": 3}[fmt], nseg, seg_len, None,
                                           out.data_ptr(), None, None, None, xs._stream_ptr(d.device))
        assert rc == 0
        assert (out.cpu().numpy().view(np.uint64) == b64).all(), (fmt, seg_len, off)
