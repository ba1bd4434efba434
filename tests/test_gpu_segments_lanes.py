"""GPU parity of K11 (one lane per segment; equal segments of length <= 256, SURVEY.md §8(f) f1
batched exact sums) in every input format: values (both roundings), flags and canonical images vs
the oracle, across the dispatch threshold, with narrow and wide exponent ranges (the touched
digit-range tracking), cancellation, specials, signed zeros and misaligned bases. Also: the
ticket-word dynamic order of ragged CSR segments (xsum_sum_segments_ws) vs the static order."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def xs():
    import torch  # noqa: F401
    import paper_1605_05436_b200 as xsum
    xsum.build()
    synth.build()
    return xsum


FMT = {"f64": (np.uint64, 0x7FF0000000000000, 64), "f32": (np.uint32, 0x7F800000, 32),
       "f16": (np.uint16, 0x7C00, 16), "bf16": (np.uint16, 0x7F80, 16)}


def data(fmt: str, n: int, seed: int, narrow: bool) -> np.ndarray:
    ut, em, bits = FMT[fmt]
    rng = np.random.default_rng(seed)
    if fmt == "f64":
        b = synth.gen.generate("c1" if narrow else "c2", seed, n).view(np.uint64).copy()
    else:
        b = rng.integers(0, 1 << bits, size=n, dtype=np.uint64).astype(ut)
        if narrow:                                       # exponent field pinned to 3 values
            t = {32: 23, 16: 10 if fmt == "f16" else 7}[bits]
            e0 = {32: 120, 16: 12 if fmt == "f16" else 120}[bits]
            e = rng.integers(e0, e0 + 3, size=n).astype(np.uint64)
            b = ((b.astype(np.uint64) & np.uint64(~em & ((1 << bits) - 1))) | (e << np.uint64(t))).astype(ut)
        fin = (b & ut(em)) == ut(em)
        b[fin] ^= ut(em & ~(em << 1) & ((1 << bits) - 1))
    k = rng.integers(0, n, size=max(1, n // 300))        # cancellation partners, zeros, specials
    b[k] = b[(k + 1) % n] ^ ut(1 << (bits - 1))
    z = rng.integers(0, n, size=max(1, n // 500))
    b[z] = ut(1 << (bits - 1))
    sp = rng.integers(0, n, size=max(1, n // 2000))
    b[sp] = np.array([em, em | (1 << (bits - 1)), em | 1], dtype=np.uint64)[rng.integers(0, 3, size=sp.size)].astype(ut)
    return b


def to_dev(b: np.ndarray, fmt: str, off: int):
    import torch
    it = {"f64": torch.int64, "f32": torch.int32, "f16": torch.int16, "bf16": torch.int16}[fmt]
    dt = {"f64": torch.float64, "f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}[fmt]
    nt = {"f64": np.int64, "f32": np.int32, "f16": np.int16, "bf16": np.int16}[fmt]
    buf = torch.empty(b.size + 8, dtype=it, device="cuda")
    t = buf[off:off + b.size]
    t.copy_(torch.from_numpy(b.view(nt)))
    return t.view(dt)


def ref(fmt, seg):
    if fmt == "f64":
        return oracle.exact_sum(seg.view(np.float64))
    if fmt == "f32":
        return oracle.exact_sum(seg.view(np.float32))
    return oracle.exact_sum(seg, fmt=fmt)


@pytest.mark.parametrize("fmt", ["f64", "f32", "f16", "bf16"])
@pytest.mark.parametrize("L", [1, 2, 3, 7, 8, 9, 33, 64, 255, 256, 257])
@pytest.mark.parametrize("narrow", [True, False])
def test_short_segments_vs_oracle(xs, fmt, L, narrow):
    nseg = 100
    b = data(fmt, nseg * L, 1000 + L, narrow)
    off = L % 3                                          # misaligned bases too (scalar-load path)
    vals, canon, flags = xs.sum_segments(to_dev(b, fmt, off), L, canon=True, flags=True)
    v = vals.cpu().numpy()
    v = v.view(np.uint64) if fmt == "f64" else v.view(np.uint32)
    cn = canon.cpu().numpy().view(np.uint64)
    fl = flags.cpu().numpy().view(np.uint32)
    for s in range(nseg):
        r, limbs = ref(fmt, b[s * L:(s + 1) * L])
        want = r.bits if fmt == "f64" else r.bits_f32
        assert int(v[s]) == want and int(fl[s]) == r.flags, (fmt, L, narrow, s)
        assert (cn[s] == limbs).all(), (fmt, L, narrow, s)
    # without images: the top-digit rounding (values with flags: the strict test; values alone)
    vals2, _, flags2 = xs.sum_segments(to_dev(b, fmt, off), L, flags=True)
    vals3, _, _ = xs.sum_segments(to_dev(b, fmt, off), L)
    assert vals2.cpu().numpy().tobytes() == vals.cpu().numpy().tobytes()
    assert flags2.cpu().numpy().tobytes() == flags.cpu().numpy().tobytes()
    assert vals3.cpu().numpy().tobytes() == vals.cpu().numpy().tobytes()


def test_short_segments_both_roundings(xs):
    """xsum_sum_segments_ex with both outputs on short binary64 segments: the binary32 rounding of
    each exact sum (one rounding) next to the binary64 one."""
    import torch
    L, nseg = 5, 1000
    b = data("f64", L * nseg, 5, False)
    d = to_dev(b, "f64", 0)
    o64 = torch.empty(nseg, dtype=torch.float64, device="cuda")
    o32 = torch.empty(nseg, dtype=torch.float32, device="cuda")
    rc = xs.lib().xsum_sum_segments_ex(d.data_ptr(), 0, nseg, L, None, o64.data_ptr(), o32.data_ptr(), None, None,
                                       torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    v64, v32 = o64.cpu().numpy().view(np.uint64), o32.cpu().numpy().view(np.uint32)
    for s in range(nseg):
        r, _ = ref("f64", b[s * L:(s + 1) * L])
        assert (int(v64[s]), int(v32[s])) == (r.bits, r.bits_f32), s


def test_ticket_and_static_order_identical(xs):
    """xsum_sum_segments_ws: ragged CSR segments with the dynamic ticket order give bit-identical
    values, flags and images to the static order (exact sums do not depend on which warp takes
    which segment); a misaligned ticket word is rejected."""
    import torch
    rng = np.random.default_rng(3)
    lens = rng.integers(0, 3000, size=700)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    for fmt in ("f64", "f32", "bf16"):
        b = data(fmt, int(offs[-1]), 77, False)
        d = to_dev(b, fmt, 0)
        o = torch.from_numpy(offs).cuda()
        st = torch.cuda.current_stream().cuda_stream
        outs = []
        for use_ticket in (False, True):
            f64 = fmt == "f64"
            out = torch.empty(lens.size, dtype=torch.float64 if f64 else torch.float32, device="cuda")
            cn = torch.empty((lens.size, 34), dtype=torch.int64, device="cuda")
            fl = torch.empty(lens.size, dtype=torch.int32, device="cuda")
            tk = torch.zeros(1, dtype=torch.int64, device="cuda")
            rc = xs.lib().xsum_sum_segments_ws(d.data_ptr(), xs._DT[str(d.dtype)[6:]], lens.size, 0, o.data_ptr(),
                                              out.data_ptr() if f64 else None, None if f64 else out.data_ptr(),
                                              cn.data_ptr(), fl.data_ptr(), tk.data_ptr() if use_ticket else None, st)
            assert rc == 0
            outs.append((out.cpu().numpy().tobytes(), cn.cpu().numpy().tobytes(), fl.cpu().numpy().tobytes()))
            if use_ticket:
                assert int(tk.item()) >= lens.size                 # the warps drew every segment
        assert outs[0] == outs[1], fmt
        for s in range(0, lens.size, 97):
            r, limbs = ref(fmt, b[offs[s]:offs[s + 1]])
            got = np.frombuffer(outs[1][0], dtype=np.uint64 if fmt == "f64" else np.uint32)[s]
            assert int(got) == (r.bits if fmt == "f64" else r.bits_f32), (fmt, s)
    tk = torch.zeros(2, dtype=torch.int64, device="cuda")
    out = torch.empty(4, dtype=torch.float64, device="cuda")
    x = torch.zeros(8, dtype=torch.float64, device="cuda")
    o = torch.tensor([0, 2, 4, 6, 8], dtype=torch.int64, device="cuda")
    assert xs.lib().xsum_sum_segments_ws(x.data_ptr(), 0, 4, 0, o.data_ptr(), out.data_ptr(), None, None, None,
                                        tk.data_ptr() + 4, torch.cuda.current_stream().cuda_stream) == xs.EINVAL


@pytest.mark.parametrize("fmt", ["f64", "f32", "f16", "bf16"])
@pytest.mark.parametrize("mix", ["short", "mixed", "empty"])
def test_csr_lanes_vs_oracle(xs, fmt, mix):
    """K11c (xsum_sum_segments_csr_lanes, picked by the binding when the mean CSR length is <= 256):
    short segments one lane each, the longer ones of a 32-segment group by the whole warp; values,
    flags and canonical images of every segment vs the oracle, misaligned starts included."""
    import torch
    rng = np.random.default_rng({"short": 1, "mixed": 2, "empty": 3}[mix])
    nseg = 1500
    lens = rng.integers(0, 40, size=nseg)
    if mix == "mixed":                                   # a few long segments (warp path), incl. > a window
        k = rng.integers(0, nseg, size=12)
        lens[k] = rng.integers(257, 70_000, size=12)
    if mix == "empty":
        lens[rng.integers(0, nseg, size=nseg // 2)] = 0
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    total = int(offs[-1])
    b = data(fmt, max(total, 1) + 300 * nseg, 40 + nseg, mix == "short")   # spare tail: mean <= 256
    d = to_dev(b, fmt, 1)
    o = torch.from_numpy(offs).cuda()
    runs = [xs.sum_segments_csr(d, o, canon=True, flags=True)]           # the binding's choice
    f64 = fmt == "f64"                                                    # and K11c explicitly
    out = torch.empty(nseg, dtype=torch.float64 if f64 else torch.float32, device="cuda")
    cnt = torch.empty((nseg, 34), dtype=torch.int64, device="cuda")
    flt = torch.empty(nseg, dtype=torch.int32, device="cuda")
    for tk in (None, torch.zeros(1, dtype=torch.int64, device="cuda")):
        rc = xs.lib().xsum_sum_segments_csr_lanes(d.data_ptr(), xs._DT[str(d.dtype)[6:]], nseg, o.data_ptr(),
                                                 out.data_ptr() if f64 else None, None if f64 else out.data_ptr(),
                                                 cnt.data_ptr(), flt.data_ptr(), tk.data_ptr() if tk is not None else None,
                                                 torch.cuda.current_stream().cuda_stream)
        assert rc == 0
        runs.append((out.clone(), cnt.clone(), flt.clone()))
    vo, _, fo = xs.sum_segments_csr(d, o, flags=True)                   # no images: top-digit rounding
    va, _, _ = xs.sum_segments_csr(d, o)
    assert vo.cpu().numpy().tobytes() == runs[0][0].cpu().numpy().tobytes()
    assert fo.cpu().numpy().tobytes() == runs[0][2].cpu().numpy().tobytes()
    assert va.cpu().numpy().tobytes() == runs[0][0].cpu().numpy().tobytes()
    for vals, canon, flags in runs:
        v = vals.cpu().numpy()
        v = v.view(np.uint64) if fmt == "f64" else v.view(np.uint32)
        cn = canon.cpu().numpy().view(np.uint64)
        fl = flags.cpu().numpy().view(np.uint32)
        for s in range(nseg):
            r, limbs = ref(fmt, b[offs[s]:offs[s + 1]])
            want = r.bits if fmt == "f64" else r.bits_f32
            assert int(v[s]) == want and int(fl[s]) == r.flags, (fmt, mix, s, lens[s])
            assert (cn[s] == limbs).all(), (fmt, mix, s)


@pytest.mark.parametrize("L", [2, 4, 6, 16, 18, 64, 256])
@pytest.mark.parametrize("narrow", [False, True])
def test_lanes_f64_values_only_paths(xs, L, narrow):
    """binary64 equal segments WITHOUT canonical images: the one-pass rounding of the raw digits
    (lane_top_fused) in both the bulk-copy kernel (L <= 16) and the prefetching one, values alone
    and values + flags, vs the oracle's per-segment sums; with exact-zero, negative, borrow-chain
    (a large term cancelled down to a tiny remainder) and special-value segments."""
    import torch
    nseg = 3001
    b = data("f64", nseg * L, 40 + L, narrow)
    x = b.view(np.float64).copy()
    # crafted segments: exact zero, a cancellation leaving a tiny negative remainder, a tie
    x[0:L] = 0.0
    x[L:2 * L] = 0.0
    x[L] = 2.0 ** 900
    x[L + 1] = -(2.0 ** 900)
    if L >= 4:
        x[L + 2] = 2.0 ** -1000
        x[L + 3] = -(2.0 ** -999)
    x[2 * L:3 * L] = 0.0
    x[2 * L] = 1.0
    x[2 * L + 1] = 2.0 ** -53
    d = torch.from_numpy(x).cuda()
    b64, _, fl, _ = oracle.sum_segments(x, seg_len=L)
    v, _, _ = xs.sum_segments(d, L)
    assert (v.cpu().numpy().view(np.uint64) == b64).all()
    v2, _, f2 = xs.sum_segments(d, L, flags=True)
    assert (v2.cpu().numpy().view(np.uint64) == b64).all()
    assert (f2.cpu().numpy().astype(np.uint32) == fl).all()


@pytest.mark.parametrize("L", [2, 8, 16, 18, 64, 256])
def test_lanes_f64_two_digit_rounding_boundaries(xs, L):
    """The values-only K11s epilogue rounds from the two top raw digits when they decide it
    (lane_fast_round) and otherwise runs the exact chain. Segments built at its decision
    boundaries: a binary64 / binary32 tie or a result one unit from a rounding or binade boundary
    in the top digits, tipped either way (or not) by tiny terms in the lower digits, with both
    signs, at exponents spread over the whole range (near overflow and where binary32 is
    subnormal or zero); values and flags (both roundings) vs the oracle."""
    import torch
    rng = np.random.default_rng(700 + L)
    nseg = 4096
    x = np.zeros((nseg, L))
    for s in range(nseg):
        e = int(rng.integers(-900, 1000))
        sg = 1.0 if rng.random() < 0.5 else -1.0
        prec = 53 if rng.random() < 0.5 else 24
        m = float(rng.integers(1 << 20, 1 << 21))             # a few significant bits at the top
        top = sg * m * 2.0 ** e
        half = 2.0 ** (e + 20 - prec) * (1 if rng.random() < 0.7 else 2)   # half an ulp (or an ulp) of top
        x[s, 0] = top
        if L >= 2:
            x[s, 1] = sg * half * (1 if rng.random() < 0.8 else -1)
        tiny_e = e - int(rng.integers(60, 300))
        for k in range(2, L):
            r = rng.random()
            x[s, k] = 0.0 if r < 0.3 else (1.0 if r < 0.65 else -1.0) * 2.0 ** (tiny_e - int(rng.integers(0, 40)))
    x = x.reshape(-1)
    x[~np.isfinite(x)] = 0.0
    d = torch.from_numpy(x).cuda()
    b64, b32, fl, _ = oracle.sum_segments(x, seg_len=L)
    v, _, f = xs.sum_segments(d, L, flags=True)
    assert (v.cpu().numpy().view(np.uint64) == b64).all()
    assert (f.cpu().numpy().astype(np.uint32) == fl).all()
    v2, _, _ = xs.sum_segments(d, L)                        # values alone (binary64 rounding only)
    assert (v2.cpu().numpy().view(np.uint64) == b64).all()


@pytest.mark.parametrize("L", [2, 8, 16, 18, 64, 256])
def test_lanes_f64_values_only_representable_tops(xs, L):
    """K11s without flags decides the rounding next to representable values from the top digits
    (lane_fast_round, need_flags false): a segment's largest element isolated 60-900 binades above
    the rest (its sum is representable up to a tail far below half an ulp), at powers of two (a
    negative tail moves the exact sum into the lower binade), at the largest mantissa, next to
    DBL_MAX (finite) and at the overflow midpoint, both signs; values alone and with flags (the
    strict test) vs the oracle."""
    import torch
    rng = np.random.default_rng(900 + L)
    nseg = 4096
    x = np.zeros((nseg, L))
    for s in range(nseg):
        kind = s % 4
        e = int(rng.integers(-800, 1000))
        sg = 1.0 if rng.random() < 0.5 else -1.0
        if kind == 0:
            top = 2.0 ** e
        elif kind == 1:
            top = (2.0 - 2.0 ** -52) * 2.0 ** min(e, 1022)
        elif kind == 2:
            top = float(rng.integers(1 << 52, 1 << 53)) * 2.0 ** (min(e, 960) - 52)
        else:
            top = np.finfo(np.float64).max
        x[s, 0] = sg * top
        if L >= 2:
            if kind == 3 and rng.random() < 0.5:
                x[s, 1] = sg * 2.0 ** 970                        # the overflow midpoint (ties to even: Inf)
            else:
                te = int(np.log2(abs(top))) - int(rng.integers(60, 900))
                for k in range(1, L):
                    r = rng.random()
                    x[s, k] = 0.0 if r < 0.2 else (1.0 if r < 0.6 else -1.0) * 2.0 ** max(te - int(rng.integers(0, 60)), -1074)
    x = x.reshape(-1)
    x[~np.isfinite(x)] = 0.0
    d = torch.from_numpy(x).cuda()
    b64, b32, fl, _ = oracle.sum_segments(x, seg_len=L)
    v, _, _ = xs.sum_segments(d, L)
    assert (v.cpu().numpy().view(np.uint64) == b64).all()
    v2, _, f = xs.sum_segments(d, L, flags=True)
    assert (v2.cpu().numpy().view(np.uint64) == b64).all()
    assert (f.cpu().numpy().astype(np.uint32) == fl).all()


@pytest.mark.parametrize("L", [5, 6, 16, 64])
def test_short_segments_tiny_sum_binary32(xs, L):
    """Regression (round 2): a segment whose exact sum is ~2^-276 with a three-digit top T of ~2^122 -
    far below binary32's least subnormal, so its binary32 rounding is -0 - rounded to the smallest
    subnormal in lane_fast_round's rounds-to-zero branch (its bound on the rounding position was 120
    where T reaches 2^126). The case came from test_short_segments_both_roundings' data (segment 383);
    it is placed in every slot of a batch of segments, zero-padded to L (K11 generic / K11s / K11)."""
    import torch
    b = data("f64", 5 * 1000, 5, False)
    base = b[383 * 5:384 * 5]
    seg = np.zeros(L, dtype=b.dtype)                               # bit patterns; zeros pad
    seg[:5] = base
    nseg = 64
    x = np.tile(seg, nseg)
    d = to_dev(x, "f64", 0)
    o64 = torch.empty(nseg, dtype=torch.float64, device="cuda")
    o32 = torch.empty(nseg, dtype=torch.float32, device="cuda")
    rc = xs.lib().xsum_sum_segments_ex(d.data_ptr(), 0, nseg, L, None, o64.data_ptr(), o32.data_ptr(), None, None,
                                       torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    r, _ = ref("f64", seg)
    assert r.bits_f32 == 0x80000000                                 # the oracle: -0 in binary32
    assert (o64.cpu().numpy().view(np.uint64) == r.bits).all()
    assert (o32.cpu().numpy().view(np.uint32) == r.bits_f32).all()
