"""GPU parity of xsum_sum_strided (K10: exact reduction along a tensor
dimension without a transposing copy): every fibre of [outer][len][inner] vs the oracle, in every
input format, both roundings and the flags; fibre counts that fill the GPU in one pass and ones
that take the split-and-merge path (same bits with and without the work buffer); ragged inner
sizes, empty reductions, specials, the per-lane rounding's edge values, argument errors."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

F_NAN, F_PINF, F_NINF = 1, 2, 4
F_OVF, F_INX, F_OVF32, F_INX32 = 8, 16, 64, 128


@pytest.fixture(scope="module")
def xs():
    import torch  # noqa: F401
    import paper_1605_05436_b200 as xsum
    xsum.build()
    synth.build()
    return xsum


def patterns(fmt: str, n: int, seed: int, specials: bool = True) -> np.ndarray:
    """Seeded bit patterns over every exponent (subnormals, zeros, both signs) plus a few NaN/Inf."""
    rng = np.random.default_rng(seed)
    if fmt == "f64":
        b = synth.gen.generate("c2", seed, n).view(np.uint64).copy()
        return _with_specials(b, rng, 0x7FF0000000000000, 64) if specials else b
    bits = 32 if fmt == "f32" else 16
    ut = np.uint32 if fmt == "f32" else np.uint16
    em = {"f32": 0x7F800000, "f16": 0x7C00, "bf16": 0x7F80}[fmt]
    b = rng.integers(0, 1 << bits, size=n, dtype=np.uint64).astype(ut)
    fin = (b & ut(em)) == ut(em)
    b[fin] ^= ut(em & ~(em << 1) & ((1 << bits) - 1))        # move the all-ones exponent down one
    return _with_specials(b, rng, em, bits) if specials else b


def _with_specials(b, rng, em, bits):
    if b.size:
        k = rng.integers(0, b.size, size=max(1, b.size // 5000))
        sign = np.array(1 << (bits - 1), dtype=np.uint64)
        vals = np.array([em, int(em) | int(sign), em | 1], dtype=np.uint64)
        b[k] = vals[rng.integers(0, 3, size=k.size)].astype(b.dtype)
    return b


def ref(fmt: str, fibre: np.ndarray):
    if fmt == "f64":
        return oracle.exact_sum(fibre.view(np.float64))
    if fmt == "f32":
        return oracle.exact_sum(fibre.view(np.float32))
    return oracle.exact_sum(fibre, fmt=fmt)


def dev(b: np.ndarray, fmt: str):
    import torch
    it = {"f64": torch.int64, "f32": torch.int32, "f16": torch.int16, "bf16": torch.int16}[fmt]
    dt = {"f64": torch.float64, "f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}[fmt]
    nt = {"f64": np.int64, "f32": np.int32, "f16": np.int16, "bf16": np.int16}[fmt]
    return torch.from_numpy(np.ascontiguousarray(b).view(nt)).cuda().view(dt)


def check(xs, fmt, b, outer, length, inner, work=True, sample=None):
    """Run xsum_sum_strided with both outputs and flags; compare fibres (all or a sample)."""
    import torch
    x = dev(b, fmt)
    F = outer * inner
    o64 = torch.empty(F, dtype=torch.float64, device="cuda")
    o32 = torch.empty(F, dtype=torch.float32, device="cuda")
    fl = torch.empty(F, dtype=torch.int32, device="cuda")
    wb = int(xs.lib().xsum_sum_strided_work_bytes(outer, length, inner, 0)) if work else 0
    wk = torch.empty(max(wb, 8), dtype=torch.uint8, device="cuda")
    rc = xs.lib().xsum_sum_strided(x.data_ptr() if x.numel() else wk.data_ptr(), xs._DT[str(x.dtype)[6:]], outer,
                                   length, inner, o64.data_ptr(), o32.data_ptr(), fl.data_ptr(),
                                   wk.data_ptr() if wb else None, wb, torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    v64 = o64.cpu().numpy().view(np.uint64)
    v32 = o32.cpu().numpy().view(np.uint32)
    f = fl.cpu().numpy().view(np.uint32)
    a3 = b.reshape(outer, length, inner) if b.size else np.zeros((outer, length, inner), dtype=b.dtype)
    idx = range(F) if sample is None else sample
    for k in idx:
        o, i = divmod(k, inner)
        r, _ = ref(fmt, np.ascontiguousarray(a3[o, :, i]))
        want_fl = r.flags & (F_NAN | F_PINF | F_NINF | F_OVF | F_INX | F_OVF32 | F_INX32)
        assert (int(v64[k]), int(v32[k]), int(f[k])) == (r.bits, r.bits_f32, want_fl), (fmt, outer, length, inner, k)
    return v64, v32, f, wb


@pytest.mark.parametrize("fmt", ["f64", "f32", "f16", "bf16"])
@pytest.mark.parametrize("outer,length,inner", [(1, 300, 37), (3, 1001, 64), (2, 5, 1000), (5, 0, 40),
                                                (1, 1, 33), (4, 2, 31)])
def test_strided_fibres_vs_oracle(xs, fmt, outer, length, inner):
    b = patterns(fmt, outer * length * inner, 100 + outer + length + inner)
    check(xs, fmt, b, outer, length, inner)


@pytest.mark.parametrize("fmt", ["f64", "f32", "bf16"])
def test_strided_split_and_merge(xs, fmt):
    """Few fibres, long reductions: the rows are split into parts merged by a second launch; the
    bits equal the oracle's and the unsplit run's (no work buffer)."""
    outer, length, inner = 1, 20_011, 70                  # 3 warps of fibres -> split into parts
    b = patterns(fmt, outer * length * inner, 7)
    v64, v32, f, wb = check(xs, fmt, b, outer, length, inner, work=True)
    assert wb > 0
    u64, u32, g, wb0 = check(xs, fmt, b, outer, length, inner, work=False)
    assert wb0 == 0 and (v64 == u64).all() and (v32 == u32).all() and (f == g).all()


def test_strided_large_sampled(xs):
    """A [4096][1024] binary64 reduction over dim 0 (one pass, many warps), sampled fibres."""
    outer, length, inner = 1, 4096, 1024
    b = patterns("f64", outer * length * inner, 9, specials=False)
    rng = np.random.default_rng(1)
    check(xs, "f64", b, outer, length, inner, sample=list(rng.integers(0, inner, size=48)) + [0, inner - 1])


def test_strided_rounding_edges(xs):
    """Per-lane canonicalization and rounding: cancellation to zero, borrows that clear the top
    digit, ties both ways, overflow, subnormal binary32 results, one fibre each."""
    vals = [
        [1.0, -1.0], [2.0 ** 1023, 1.0, -(2.0 ** 1023)], [1.0, 2.0 ** -53], [1.0, 2.0 ** -52, 2.0 ** -53],
        [1.7976931348623157e308, 2.0 ** 970], [1.7976931348623157e308, 2.0 ** 969], [-0.0, -0.0],
        [2.0 ** 104, -1.0], [-(2.0 ** 104), 1.0], [2.0 ** -1074, 2.0 ** -1074], [2.0 ** -150, 2.0 ** -160],
        [-(2.0 ** -150)], [3.4028235677973366e38, 1.0e30], [1.0 + 2.0 ** -23, 2.0 ** -24, 2.0 ** -60],
        [2.0 ** 127, 2.0 ** 127], [-(2.0 ** 128)],               # exact sums that overflow binary32
    ]
    length = max(len(v) for v in vals)
    inner = len(vals)
    a = np.zeros((length, inner))
    for i, v in enumerate(vals):
        a[:len(v), i] = v
    check(xs, "f64", a.reshape(-1).view(np.uint64).copy(), 1, length, inner)


def test_exact_sum_dim_uses_strided_path(xs):
    """exact_sum_dim over a non-last dimension of a contiguous tensor (the strided kernel) and of a
    non-contiguous view (movedim + segments) give the oracle's bits."""
    import torch
    x = synth.gen.generate("c2", 21, 6 * 500 * 70).reshape(6, 500, 70)
    t = torch.from_numpy(x).cuda()
    for dim, tt in ((1, t), (0, t), (1, t.transpose(0, 2))):
        out = xs.exact_sum_dim(tt, dim).cpu().numpy()
        xx = tt.cpu().numpy()
        fib = np.moveaxis(xx, dim, -1).reshape(-1, xx.shape[dim])
        for k in range(0, fib.shape[0], max(1, fib.shape[0] // 40)):
            r, _ = oracle.exact_sum(fib[k])
            assert out.reshape(-1)[k].view(np.uint64) == np.uint64(r.bits), (dim, k)


def test_strided_argument_errors(xs):
    import torch
    L = xs.lib()
    x = torch.zeros(64, dtype=torch.float64, device="cuda")
    o = torch.zeros(8, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    assert L.xsum_sum_strided(x.data_ptr(), 9, 1, 8, 8, o.data_ptr(), None, None, None, 0, st) == xs.EINVAL
    assert L.xsum_sum_strided(x.data_ptr(), 0, 1, 8, 8, None, None, None, None, 0, st) == xs.EINVAL
    assert L.xsum_sum_strided(x.data_ptr() + 4, 0, 1, 8, 8, o.data_ptr(), None, None, None, 0, st) == xs.EINVAL
    assert L.xsum_sum_strided(x.data_ptr(), 0, 0, 8, 8, o.data_ptr(), None, None, None, 0, st) == 0
    assert L.xsum_sum_strided(x.data_ptr(), 0, 1 << 62, 8, 8, o.data_ptr(), None, None, None, 0, st) == xs.EINVAL


@pytest.mark.parametrize("shape,perm,dim", [((300, 70), (1, 0), 1), ((300, 70), (1, 0), 0), ((6, 50, 70), (2, 0, 1), 2),
                                            ((6, 50, 70), (1, 2, 0), 0), ((4, 1, 90), (2, 1, 0), 2)])
def test_exact_sum_dim_permuted_views(xs, shape, perm, dim):
    """exact_sum_dim of a permuted (e.g. transposed) view of a contiguous tensor: the matching
    dimension of the underlying layout is reduced in place and the output put back in the view's
    order; every fibre vs the oracle."""
    import torch
    n = int(np.prod(shape))
    x = synth.gen.generate("c2", 31, n).reshape(shape)
    t = torch.from_numpy(x).cuda().permute(perm)
    assert not t.is_contiguous() or shape[1] == 1
    out = xs.exact_sum_dim(t, dim).cpu().numpy()
    xv = np.transpose(x, perm)
    assert out.shape == np.sum(xv, axis=dim).shape
    fib = np.moveaxis(xv, dim, -1).reshape(-1, xv.shape[dim])
    for k in range(fib.shape[0]):
        r, _ = oracle.exact_sum(np.ascontiguousarray(fib[k]))
        assert out.reshape(-1)[k].view(np.uint64) == np.uint64(r.bits), (shape, perm, dim, k)
    kd = xs.exact_sum_dim(t, dim, keepdim=True)
    assert tuple(kd.shape) == tuple(np.sum(xv, axis=dim, keepdims=True).shape)


@pytest.mark.parametrize("shape,dim", [((6, 50, 70), (1, 2)), ((6, 50, 70), (0, 1)), ((6, 50, 70), (0, 2)),
                                       ((6, 50, 70), (-1, 0, 1)), ((6, 50, 70), None), ((5,), None)])
def test_exact_sum_dim_tuples_and_none(xs, shape, dim):
    """exact_sum_dim with a tuple of dimensions (adjacent: merged without a copy; otherwise moved
    last) or None (everything; a 0-d device tensor): the oracle's exact sums, keepdim shapes."""
    import torch
    n = int(np.prod(shape))
    x = synth.gen.generate("c2", 41, n).reshape(shape)
    t = torch.from_numpy(x).cuda()
    out = xs.exact_sum_dim(t, dim)
    ref_shape = np.sum(x, axis=None if dim is None else tuple(dim)).shape
    assert tuple(out.shape) == tuple(ref_shape)
    o = out.cpu().numpy().reshape(-1)
    if dim is None:
        r, _ = oracle.exact_sum(x.reshape(-1))
        assert o[0:1].view(np.uint64)[0] == np.uint64(r.bits)
    else:
        dims = sorted({k % len(shape) for k in dim})
        keep = [k for k in range(len(shape)) if k not in dims]
        fib = np.transpose(x, keep + dims).reshape(o.size, -1)
        for k in range(o.size):
            r, _ = oracle.exact_sum(np.ascontiguousarray(fib[k]))
            assert o[k:k + 1].view(np.uint64)[0] == np.uint64(r.bits), (dim, k)
    kd = xs.exact_sum_dim(t, dim, keepdim=True)
    assert tuple(kd.shape) == tuple(np.sum(x, axis=None if dim is None else tuple(dim), keepdims=True).shape)
    # a narrow format with dim=None gives the binary32 rounding of the exact sum
    b = synth.gen.bits("c2bf16", 0, 1001)
    tb = torch.from_numpy(b.view(np.int16)).cuda().view(torch.bfloat16)
    r, _ = oracle.exact_sum(b, fmt="bf16")
    assert xs.exact_sum_dim(tb, None).cpu().numpy().reshape(1).view(np.uint32)[0] == r.bits_f32


@pytest.mark.parametrize("fmt", ["f16", "bf16"])
@pytest.mark.parametrize("outer,length,inner", [(2, 5000, 96), (1, 1537, 130), (3, 513, 2), (1, 70_001, 64)])
def test_strided_h16_two_fibres_per_lane(xs, fmt, outer, length, inner):
    """K10h (16-bit, even inner, 4-B aligned base: two fibres per lane, packed decode into bins):
    reductions longer than a bin window (bfloat16: 512 rows), inner sizes that end mid-warp, the
    split path (with and without the work buffer) - every fibre vs the oracle."""
    b = patterns(fmt, outer * length * inner, 900 + length + inner)
    v64, v32, f, wb = check(xs, fmt, b, outer, length, inner, work=True)
    u64, u32, g, _ = check(xs, fmt, b, outer, length, inner, work=False, sample=range(min(40, outer * inner)))
    assert (v64[:40] == u64[:40]).all() and (v32[:40] == u32[:40]).all()


def test_strided_h16_misaligned_base_falls_back(xs):
    """A base that is not 4-B aligned takes the one-fibre-per-lane kernel: same bits."""
    import torch
    b = patterns("bf16", 1 + 700 * 64, 31)
    x = dev(b, "bf16")[1:].view(700, 64)
    assert x.data_ptr() % 4 == 2
    out = xs.exact_sum_dim(x, 0).cpu().numpy().view(np.uint32)
    a = b[1:].reshape(700, 64)
    for i in range(64):
        r, _ = ref("bf16", np.ascontiguousarray(a[:, i]))
        assert int(out[i]) == r.bits_f32


@pytest.mark.parametrize("fmt", ["f64", "f32", "bf16"])
def test_strided_split_many_fibres(xs, fmt):
    """Many fibres that still under-fill the GPU: the rows are split into parts and the parts are
    merged one lane per fibre (k_strided_merge_lanes); every fibre vs the oracle's per-fibre sums."""
    import torch
    length, inner = 1536, 40_000
    b = patterns(fmt, length * inner, 4242)
    wb = int(xs.lib().xsum_sum_strided_work_bytes(1, length, inner, 0))
    assert wb > 0                                           # the split path is taken
    x = dev(b, fmt).view(length, inner)
    out = xs.exact_sum_dim(x, 0)
    got = out.cpu().numpy().view(np.uint64 if fmt == "f64" else np.uint32)
    host_t = np.ascontiguousarray(b.reshape(length, inner).T).reshape(-1)
    if fmt == "f32":
        host_t = host_t.view(np.float32)
    b64, b32, _, _ = oracle.sum_segments(host_t, seg_len=length, fmt=fmt if fmt in ("f16", "bf16") else None)
    assert (got == (b64 if fmt == "f64" else b32)).all()


@pytest.mark.parametrize("fmt", ["f64", "f32", "f16", "bf16"])
@pytest.mark.parametrize("outer,length,inner", [(1, 2048, 4096), (3, 777, 1000), (1, 100_003, 32)])
def test_strided_stream_k(xs, fmt, outer, length, inner):
    """K10s (fibre groups that fill the resident warps unevenly; K10 / K10f / K10h pieces): every warp
    takes an equal share of all rows, so fibres are split across 1-3 warps (or, for few long fibres,
    across many) whose pieces meet in the per-fibre accumulator; NaN / Inf planted in split fibres.
    Every fibre vs the oracle, and the same bits without a work buffer (the plain per-fibre kernel)."""
    b = patterns(fmt, outer * length * inner, 31 + length)
    v64, v32, f, wb = check(xs, fmt, b, outer, length, inner, work=True)
    assert wb > 0
    u64, u32, g, _ = check(xs, fmt, b, outer, length, inner, work=False,
                           sample=list(range(0, outer * inner, 97)))
    assert (v64 == u64).all() and (v32 == u32).all() and (f == g).all()
