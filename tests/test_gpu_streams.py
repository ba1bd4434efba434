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
