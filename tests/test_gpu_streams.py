"""Stream semantics of the C-ABI (include/xsum.h: calls are asynchronous and stream-ordered, one
handle per stream at a time, different handles independent) and CUDA-graph capture of the fused
one-launch sum: results vs the oracle."""
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


def test_handles_on_concurrent_streams(xs):
    import torch
    a = synth.gen.generate("c2", 21, 3_000_001)
    b = synth.gen.generate("c3", 0, 2_000_003, permute=False)
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    acc1, acc2 = xs.Accumulator(), xs.Accumulator()
    torch.cuda.synchronize()
    for _ in range(3):                                   # interleaved launches on two streams
        with torch.cuda.stream(s1):
            r1, c1 = acc1.sum(da, canon=True)
        with torch.cuda.stream(s2):
            r2, c2 = acc2.sum(db, canon=True)
    torch.cuda.synchronize()
    for res, canon, x in ((r1, c1, a), (r2, c2, b)):
        ref, limbs = oracle.exact_sum(x)
        r = xs.Result.from_bytes(res.cpu().numpy().tobytes())
        assert r.bits == ref.bits and (canon.cpu().numpy().view(np.uint64) == limbs).all()


def test_stream_ordering_of_chunked_calls(xs):
    """accumulate / merge / finalize enqueued on a side stream right after the producer of the
    data: stream order alone makes the result exact."""
    import torch
    x = synth.gen.generate("c2", 22, 4_000_000)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        d = torch.from_numpy(x).to("cuda", non_blocking=False)
        d2 = d * 1.0                                     # produced on s
        acc = xs.Accumulator()
        acc.add(d2[:1_000_000]).add(d2[1_000_000:])
        res, canon = acc.finalize_async(canon=True)
    s.synchronize()
    ref, limbs = oracle.exact_sum(x)
    r = xs.Result.from_bytes(res.cpu().numpy().tobytes())
    assert r.bits == ref.bits and (canon.cpu().numpy().view(np.uint64) == limbs).all()


def test_cuda_graph_capture_of_fused_sum(xs):
    """The fused one-launch sum captured in a CUDA graph and replayed on new input contents."""
    import torch
    n = 1_000_003
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    acc = xs.Accumulator()
    s = torch.cuda.Stream()
    d.copy_(torch.from_numpy(synth.gen.generate("c2", 30, n)))
    with torch.cuda.stream(s):
        acc.sum(d)                                       # warm (attributes set outside capture)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        res, canon = acc.sum(d, canon=True)
    for seed in (31, 32, 33):
        x = synth.gen.generate("c2", seed, n)
        d.copy_(torch.from_numpy(x))
        g.replay()
        torch.cuda.synchronize()
        ref, limbs = oracle.exact_sum(x)
        r = xs.Result.from_bytes(res.cpu().numpy().tobytes())
        assert r.bits == ref.bits and (canon.cpu().numpy().view(np.uint64) == limbs).all(), seed


def test_one_shot_helpers_per_stream(xs):
    """exact_sum_dim(dim=None) / fsum on two streams back to back: each stream has its own default
    handle (no shared scratch/state), so both device results are the oracle's."""
    import numpy as np
    import torch

    import oracle
    import synth
    a = synth.gen.generate("c2", 51, 3_000_001)
    b = synth.gen.generate("c2", 52, 2_000_003)
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        ra = xs.exact_sum_dim(da, None)
    with torch.cuda.stream(s2):
        rb = xs.exact_sum_dim(db, None)
    torch.cuda.synchronize()
    assert ra.cpu().numpy().reshape(1).view(np.uint64)[0] == oracle.exact_sum(a)[0].bits
    assert rb.cpu().numpy().reshape(1).view(np.uint64)[0] == oracle.exact_sum(b)[0].bits


def test_cuda_graph_capture_of_segment_strided_condsens_paths(xs):
    """One CUDA graph holding the other hot paths - equal segments (values + flags), a strided
    reduction over dim 0 (row-split parts + merge), the condition-number-sensitive sum and a
    binary16 fused sum - replayed on new input contents; every output vs the oracle. No call in
    these paths synchronizes with the host, so all of them are capturable."""
    import torch

    from oracle import condsens as cs
    nseg, L = 777, 1000
    rows, cols = 5000, 96
    d_seg = torch.empty(nseg * L, dtype=torch.float64, device="cuda")
    d_mat = torch.empty(rows * cols, dtype=torch.float64, device="cuda")
    d_cs = torch.empty(20_001, dtype=torch.float64, device="cuda")
    d_h = torch.empty(300_007, dtype=torch.int16, device="cuda")

    def fill(seed):
        xs_ = synth.gen.generate("c2", seed, nseg * L)
        xm = synth.gen.generate("c5", seed, rows * cols)
        xc = synth.gen.generate("c3", 2 * seed, 20_001, permute=False)
        rng = np.random.default_rng(seed)
        hb = rng.integers(-32768, 32767, size=300_007, dtype=np.int64).astype(np.int16)
        hb = np.where((hb & 0x7C00) == 0x7C00, hb ^ 0x400, hb).astype(np.int16)
        d_seg.copy_(torch.from_numpy(xs_))
        d_mat.copy_(torch.from_numpy(xm))
        d_cs.copy_(torch.from_numpy(xc))
        d_h.copy_(torch.from_numpy(hb))
        return xs_, xm, xc, hb

    s = torch.cuda.Stream()
    acc = xs.Accumulator()
    fill(60)
    torch.cuda.synchronize()

    def step():
        v, _, f = xs.sum_segments(d_seg, L, flags=True)
        m = xs.exact_sum_dim(d_mat.view(rows, cols), 0)
        r, info, _ = xs.sum_condsens(d_cs, 1)
        h, _ = acc.sum(d_h.view(torch.float16))
        return v, f, m, r, info, h

    with torch.cuda.stream(s):
        step()                                           # warm: kernel attributes, allocator
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        outs = step()
    for seed in (61, 62):
        xs_, xm, xc, hb = fill(seed)
        g.replay()
        torch.cuda.synchronize()
        v, f, m, r, info, h = outs
        b64, _, fl, _ = oracle.sum_segments(xs_, seg_len=L)
        assert (v.cpu().numpy().view(np.uint64) == b64).all() and (f.cpu().numpy().astype(np.uint32) == fl).all()
        mt = np.ascontiguousarray(xm.reshape(rows, cols).T).reshape(-1)
        bm, _, _, _ = oracle.sum_segments(mt, seg_len=rows)
        assert (m.cpu().numpy().view(np.uint64) == bm).all()
        o = cs.condsens_sum(list(xc), rule=1)
        res = xs.Result.from_bytes(r.cpu().numpy().tobytes())
        inf = xs.CondSensInfo.from_bytes(info.cpu().numpy().tobytes())
        assert inf.r == o.r and inf.iterations == o.iterations
        assert res.bits == np.float64(o.value).view(np.uint64)
        rh, _ = oracle.exact_sum(hb.view(np.uint16), fmt="f16")
        assert xs.Result.from_bytes(h.cpu().numpy().tobytes()).bits == rh.bits
