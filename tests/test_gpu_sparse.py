"""GPU parity for sparse state images (the paper's sparse superaccumulator,
PAPER.md:682-696): encode -> host decode -> exact value vs the oracle; encode -> merge round
trip; shard merges of sparse images vs the oracle; malformed images rejected."""
from __future__ import annotations

import struct

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


def dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()


def value_of(d: dict) -> int:
    return sum(v << (52 * j) for j, v in d["digits"].items())


@pytest.mark.parametrize("cfg,n", [("c1", 100_000), ("c2", 300_001), ("c3", 0), ("c5", 65536)])
def test_sparse_encode_value_and_round_trip(xs, cfg, n):
    x = synth.gen.generate(cfg, 3, n) if n else np.zeros(0)
    acc = xs.Accumulator().add(dev(x)) if n else xs.Accumulator()
    img, nb = acc.to_sparse()
    d = xs.decode_sparse(img.cpu().numpy().tobytes())
    r, limbs = oracle.exact_sum(x)
    assert value_of(d) == oracle.limbs_to_int(limbs)                      # exact value (oracle)
    assert d["count"] == n and nb == 24 + 8 * len(d["digits"])
    dense = np.frombuffer(acc.state.cpu().numpy().tobytes()[24:24 + 8 * 42], dtype="<i8")
    assert sorted(d["digits"]) == [j for j in range(42) if dense[j] != 0]  # active indices only
    if cfg == "c1":
        assert len(d["digits"]) <= 4                                       # narrow exponents: tiny image
    import torch
    b = xs.Accumulator().merge_sparse(img.clone(), torch.zeros(1, dtype=torch.int64, device="cuda"))
    assert bytes(b.state.cpu().numpy()) == bytes(acc.state.cpu().numpy())   # digit-for-digit
    assert b.result().bits == r.bits


def test_sparse_shard_merge_equals_whole(xs):
    import torch
    x = synth.gen.generate("c2", 9, 1_000_003)
    cuts = [0, 1, 77, 50_000, 400_000, 999_999, 1_000_003]
    imgs, offs, off = [], [], 0
    for a, b in zip(cuts, cuts[1:]):
        img, nb = xs.Accumulator().add(dev(x[a:b])).to_sparse()
        imgs.append(img.cpu().numpy())
        offs.append(off)
        off += nb
    blob = torch.from_numpy(np.concatenate(imgs)).cuda()
    acc = xs.Accumulator().merge_sparse(blob, torch.tensor(offs, dtype=torch.int64, device="cuda"))
    res, canon = acc.exact()
    r, limbs = oracle.exact_sum(x)
    assert res.bits == r.bits and (canon == limbs).all() and res.count == x.size and res.flags == r.flags


def test_sparse_rejects_malformed_images(xs):
    import torch
    good = struct.pack("<IHBBIIQ", 0x41505358, 1, 52, 1, 0, 0, 1) + struct.pack("<q", (5 << 6) | 21)
    bad = [
        struct.pack("<IHBBIIQ", 0x41505359, 1, 52, 1, 0, 0, 1) + struct.pack("<q", (5 << 6) | 21),   # magic
        struct.pack("<IHBBIIQ", 0x41505358, 1, 51, 1, 0, 0, 1) + struct.pack("<q", (5 << 6) | 21),   # width
        struct.pack("<IHBBIIQ", 0x41505358, 1, 52, 43, 0, 0, 1) + b"\0" * 8 * 43,                    # nnz > D
        struct.pack("<IHBBIIQ", 0x41505358, 1, 52, 2, 0, 0, 1) + struct.pack("<qq", (5 << 6) | 21, (5 << 6) | 20),
        struct.pack("<IHBBIIQ", 0x41505358, 1, 52, 1, 0, 0, 1) + struct.pack("<q", (5 << 6) | 42),   # index
        struct.pack("<IHBBIIQ", 0x41505358, 1, 52, 1, 0, 0, 1) + struct.pack("<q", ((1 << 52) << 6) | 3),
    ]
    for b in bad:
        blob = torch.from_numpy(np.frombuffer(good + b, dtype=np.uint8).copy()).cuda()
        acc = xs.Accumulator().merge_sparse(blob, torch.tensor([0, len(good)], dtype=torch.int64, device="cuda"))
        r = acc.result()
        assert r.flags & xs.F_MISMATCH and r.count == 1, b[:8]
        assert r.value == 5 * 2.0 ** (52 * 21 - 1074)            # the good image was merged
    # misaligned offset
    blob = torch.from_numpy(np.frombuffer(good + b"\0" * 4 + good, dtype=np.uint8).copy()).cuda()
    r = xs.Accumulator().merge_sparse(blob, torch.tensor([0, len(good) + 4], dtype=torch.int64,
                                                         device="cuda")).result()
    assert r.flags & xs.F_MISMATCH


@pytest.mark.parametrize("nimg", [17, 33, 48, 1000])
def test_sparse_merge_many_images_with_bad_ones(xs, nimg):
    """More images than the merge kernel's 16 leaf warps: every warp folds several images through
    its pipelined offset / header / record loads (offsets two images ahead, headers one ahead).
    Malformed images and a misaligned offset sit at positions the pipeline reaches from the
    previous iterations; the good images' exact sum and count must match the oracle."""
    import torch
    rng = np.random.default_rng(nimg)
    x = synth.gen.generate("c1", 11, 40 * nimg + 7)
    cuts = np.sort(rng.integers(0, x.size, nimg - 1))
    cuts = np.concatenate([[0], cuts, [x.size]])
    bad_hdr = struct.pack("<IHBBIIQ", 0x41505359, 1, 52, 1, 0, 0, 1) + struct.pack("<q", (5 << 6) | 21)
    bad_pos = {p for p in (16, 20, 45, 70, 999) if p < nimg}
    mis_pos = 37 if nimg > 37 else None
    parts, offs, off, good = [], [], 0, []
    for i, (a, b) in enumerate(zip(cuts, cuts[1:])):
        if i in bad_pos:
            parts.append(np.frombuffer(bad_hdr, dtype=np.uint8))
            offs.append(off)
            off += len(bad_hdr)
            continue
        img, nb = xs.Accumulator().add(dev(x[a:b])).to_sparse()
        if i == mis_pos:                                 # a 4-byte gap: this image's offset is misaligned
            parts.append(np.zeros(4, dtype=np.uint8))
            off += 4
        else:
            good.append(x[a:b])
        parts.append(img.cpu().numpy())
        offs.append(off)
        off += nb
        if i == mis_pos:                                 # realign the following images
            parts.append(np.zeros(4, dtype=np.uint8))
            off += 4
    blob = torch.from_numpy(np.concatenate(parts)).cuda()
    acc = xs.Accumulator().merge_sparse(blob, torch.tensor(offs, dtype=torch.int64, device="cuda"))
    res, canon = acc.exact()
    g = np.concatenate(good)
    r, limbs = oracle.exact_sum(g)
    assert res.bits == r.bits and (canon == limbs).all() and res.count == g.size
    assert bool(res.flags & xs.F_MISMATCH) == bool(bad_pos or mis_pos is not None)
