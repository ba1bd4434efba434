"""Full-size parity of the NEXT-row bench workloads, in the launch
configuration bench.py times: every output of the step against the oracle's per-segment sums
(oracle.sum_segments, pinned against O2 in tests/test_oracle_pins.py).

  c5csr  : 2^16 CSR segments of 1..8192 doubles      -> xsum_sum_segments_ws (warp per segment, ticket)
  c5s16  : 2^24 segments of 16 doubles               -> K11 (one lane per segment)
  c2dim0 : c2 as [4096, 65536], exact_sum_dim(dim=0) -> K10 (strided, one lane per fibre)
  c5     : 2^16 x 4096 doubles (BASELINE config 5)   -> K6h (half a warp per segment)
Values are compared bit for bit (binary64), flags and canonical images where the step returns them."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def xs():
    import torch  # noqa: F401
    import paper_1605_05436_b200 as xsum
    xsum.build()
    synth.build()
    return xsum


def test_c5csr_full(xs):
    cfg = synth.CONFIGS["c5csr"]
    d = synth.device_generate("c5csr")
    offs_d = synth.csr_offsets("c5csr", device="cuda")
    vals, canon, flags = xs.sum_segments_csr(d, offs_d, canon=True, flags=True)
    off = synth.gen.csr_offsets(cfg).astype(np.uint64)
    b64, _, fl, cn = oracle.sum_segments(synth.host_generate("c5csr"), off, canon=True)
    assert (vals.cpu().numpy().view(np.uint64) == b64).all()
    assert (flags.cpu().numpy().astype(np.uint32) == fl).all()
    assert (canon.cpu().numpy().view(np.uint64) == cn).all()


def test_c5s16_full(xs):
    cfg = synth.CONFIGS["c5s16"]
    d = synth.device_generate("c5s16")
    vals, _, flags = xs.sum_segments(d, cfg["seg_len"], flags=True)
    host = synth.host_generate("c5s16")
    b64, _, fl, _ = oracle.sum_segments(host, seg_len=cfg["seg_len"])
    assert vals.numel() == cfg["nseg"]
    assert (vals.cpu().numpy().view(np.uint64) == b64).all()
    assert (flags.cpu().numpy().astype(np.uint32) == fl).all()
    # canonical images on a prefix of 2^16 segments (the whole set would be 4.5 GB)
    k = 1 << 16
    _, canon, _ = xs.sum_segments(d[: k * 16], 16, canon=True)
    _, _, _, cn = oracle.sum_segments(host[: k * 16], seg_len=16, canon=True)
    assert (canon.cpu().numpy().view(np.uint64) == cn).all()


def test_c2dim0_full(xs):
    cfg = synth.CONFIGS["c2dim0"]
    rows, cols = cfg["shape"]
    d = synth.device_generate("c2").view(rows, cols)
    out = xs.exact_sum_dim(d, 0)
    assert tuple(out.shape) == (cols,)
    host_t = np.ascontiguousarray(synth.host_generate("c2").reshape(rows, cols).T)
    b64, _, _, _ = oracle.sum_segments(host_t.reshape(-1), seg_len=rows)
    assert (out.cpu().numpy().view(np.uint64) == b64).all()


def test_c5_full_against_batched_oracle(xs):
    cfg = synth.CONFIGS["c5"]
    d = synth.device_generate("c5")
    vals, canon, flags = xs.sum_segments(d, cfg["seg_len"], canon=True, flags=True)
    b64, _, fl, cn = oracle.sum_segments(synth.host_generate("c5"), seg_len=cfg["seg_len"], canon=True)
    assert (vals.cpu().numpy().view(np.uint64) == b64).all()
    assert (flags.cpu().numpy().astype(np.uint32) == fl).all()
    assert (canon.cpu().numpy().view(np.uint64) == cn).all()
