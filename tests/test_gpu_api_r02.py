"""GPU tests of the round-2 boundary fixes:

* xsum_count / Accumulator.count after merges (the merged count, not the host-side 0), after
  dist.allreduce_exact, and the saturating XSUM_F_CAPACITY flag when merged counts pass 2^63-1;
* one top-digit bound (|digit[41]| <= 2^29, the value bound of DESIGN.md R7) in k_merge, the
  sparse merge and xsum_check_state_image;
* tensors on another device than the accumulator raise ValueError before any launch;
* programmatic dependent launch: an accumulate launched right after a kernel that WRITES its
  input reads the written values (griddepcontrol.wait before the first input load);
* add_host keeps every pinned source alive until its copies are done.
Values are compared with the oracle (oracle/), never with the CUDA path itself."""
from __future__ import annotations

import struct

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

R = 1 << 52


@pytest.fixture(scope="module")
def xs():
    import torch  # noqa: F401
    import paper_1605_05436_b200 as xsum
    xsum.build()
    synth.build()
    return xsum


def dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def image(digits: dict, count: int = 0, flags: int = 0) -> bytes:
    """A 384-byte state image (include/xsum.h layout) built on the host."""
    d = [0] * 42
    for k, v in digits.items():
        d[k] = v
    return struct.pack("<IHBBIIQ42q", 0x4D555358, 1, 52, 42, flags, 0, count, *d) + bytes(24)


def test_count_after_merge_and_allreduce(xs):
    import torch
    x = synth.gen.generate("c2", 3, 300_001)
    d = dev(x)
    a = xs.Accumulator().add(d[:100_000])
    b = xs.Accumulator().add(d[100_000:])
    m = xs.Accumulator().merge(torch.cat([a.state, b.state]))
    assert m.count == x.size                          # the merged count, resolved from the device
    m.add(d[:5])                                      # accumulate after a merge: host adds on top
    assert m.count == x.size + 5
    m.reset()
    assert m.count == 0
    r, limbs = oracle.exact_sum(x)
    mr = xs.Accumulator().merge_round(torch.cat([a.state, b.state]))
    res = xs.Result.from_bytes(mr[0].cpu().numpy().tobytes())
    assert res.bits == r.bits and res.count == x.size


def test_count_after_allreduce_exact_gloo_world1(xs, tmp_path):
    import torch
    import torch.distributed as tdist
    from paper_1605_05436_b200 import dist
    if tdist.is_initialized():
        pytest.skip("a process group is already initialised")
    tdist.init_process_group("gloo", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1)
    try:
        x = dev(synth.gen.generate("c1", 0, 12_345))
        acc = xs.Accumulator().add(x)
        dist.allreduce_exact(acc)
        assert acc.count == 12_345
    finally:
        tdist.destroy_process_group()


def test_merged_count_saturates_with_capacity_flag(xs):
    import torch
    big = (1 << 62) + 5
    ims = image({3: 7}, count=big) + image({3: 9}, count=big)
    st = torch.from_numpy(np.frombuffer(ims, dtype=np.uint8).copy()).cuda()
    m = xs.Accumulator().merge(st)
    res = m.result()
    assert res.flags & xs.F_CAPACITY and res.count == (1 << 63) - 1
    assert res.value == 16 * 2.0 ** (-1074 + 3 * 52)     # digits stay exact
    assert m.count == (1 << 63) - 1
    assert not xs.check_state_image(m.save_state())        # not a valid checkpoint any more
    # below the limit: no flag, exact count
    ok = image({0: 1}, count=(1 << 62)) + image({0: 1}, count=(1 << 62) - 1)
    m2 = xs.Accumulator().merge(torch.from_numpy(np.frombuffer(ok, dtype=np.uint8).copy()).cuda())
    r2 = m2.result()
    assert not r2.flags & xs.F_CAPACITY and r2.count == (1 << 63) - 1


@pytest.mark.parametrize("top,accepted", [(1 << 29, True), (-(1 << 29), True), ((1 << 29) + 1, False),
                                          (-(1 << 29) - 1, False), (1 << 40, False)])
def test_one_top_digit_bound(xs, top, accepted):
    import torch
    im = image({41: top, 0: 3}, count=1)
    assert xs.check_state_image(im) == accepted
    m = xs.Accumulator().merge(torch.from_numpy(np.frombuffer(im, dtype=np.uint8).copy()).cuda())
    res = m.result()
    assert bool(res.flags & xs.F_MISMATCH) == (not accepted)
    # the same digits as a sparse image
    hdr = struct.pack("<IHBBIIQ", 0x41505358, 1, 52, 2, 0, 0, 1)
    rec = struct.pack("<qq", (3 << 6) | 0, (top << 6) | 41)
    sp = torch.from_numpy(np.frombuffer(hdr + rec, dtype=np.uint8).copy()).cuda()
    offs = torch.zeros(1, dtype=torch.int64, device="cuda")
    rs = xs.Accumulator().merge_sparse(sp, offs).result()
    assert bool(rs.flags & xs.F_MISMATCH) == (not accepted)


def test_image_with_too_large_count_rejected_by_merge(xs):
    import torch
    im = image({0: 1}, count=1 << 63)
    assert not xs.check_state_image(im)
    r = xs.Accumulator().merge(torch.from_numpy(np.frombuffer(im, dtype=np.uint8).copy()).cuda()).result()
    assert r.flags & xs.F_MISMATCH


def test_wrong_device_raises(xs):
    import torch
    if torch.cuda.device_count() < 2:
        # one GPU: a CPU tensor must still be refused before any launch
        acc = xs.Accumulator()
        with pytest.raises(TypeError):
            acc.add(torch.zeros(4, dtype=torch.float64))
        return
    acc = xs.Accumulator("cuda:0")
    other = torch.zeros(16, dtype=torch.float64, device="cuda:1")
    for call in (lambda: acc.add(other), lambda: acc.sum(other),
                 lambda: acc.merge(torch.zeros(384, dtype=torch.uint8, device="cuda:1"))):
        with pytest.raises(ValueError):
            call()


def test_on_device_check_messages(xs):
    """The device check itself (exercised with a fake tensor-like object on one GPU)."""
    import torch
    acc = xs.Accumulator()

    class Fake:
        device = torch.device("cuda", acc._idx + 1)
    with pytest.raises(ValueError):
        acc._on_device(Fake(), "x")


def test_pdl_reads_input_written_by_preceding_kernel(xs):
    """A producer kernel writes the input, an accumulate follows immediately on the same stream
    (no host sync): the sum must be of the written values, for every size class that launches
    with PDL (< 1 GiB), many times over."""
    import torch
    for n in (1 << 12, 1 << 18, (1 << 22) + 3):
        x = synth.gen.generate("c2", 11, n)
        src = dev(x)
        r, limbs = oracle.exact_sum(x)
        buf = torch.zeros_like(src)
        acc = xs.Accumulator()
        for _ in range(20):
            buf.zero_()
            res0, _ = acc.sum(buf)                   # previous accumulate launch (PDL predecessor)
            buf.copy_(src)                           # a non-xsum kernel writes the input
            res, canon = acc.sum(buf, canon=True)    # launched right behind the copy kernel
            got = xs.Result.from_bytes(res.cpu().numpy().tobytes())
            assert got.bits == r.bits and (canon.cpu().numpy().view(np.uint64) == limbs).all()


def test_add_host_keeps_sources_alive(xs):
    import gc

    import torch
    parts = [synth.gen.generate("c2", 20 + k, 1 << 18) for k in range(4)]
    r, limbs = oracle.exact_sum(np.concatenate(parts))
    acc = xs.Accumulator()
    for p in parts:
        h = torch.from_numpy(p.copy()).pin_memory()
        acc.add_host(h, stage_bytes=2 << 20)
        del h
        gc.collect()
        # reuse pinned memory immediately: a freed source block must not be handed out while
        # its copies are pending
        junk = torch.full((1 << 18,), float("nan"), dtype=torch.float64).pin_memory()
        del junk
    res, canon = acc.exact()
    assert res.bits == r.bits and (canon == limbs).all()
    assert len(acc._host_refs) <= 4


def test_one_shot_cache_bounded(xs):
    import torch
    x = dev(synth.gen.generate("c1", 0, 1000))
    want = xs.fsum(x)
    streams = [torch.cuda.Stream() for _ in range(40)]
    for s in streams:
        with torch.cuda.stream(s):
            assert xs.fsum(x) == want
    assert len(xs._default_acc) <= xs._DEFAULT_ACC_MAX


def test_pdl_consumer_waits_for_an_early_triggering_producer(xs):
    """a producer that releases its programmatic dependents BEFORE writing the
    input (synth's k_fill_after_trigger: 4 blocks, launch_dependents, ~100 us spin, then the stores)
    directly followed by PDL-launched accumulate kernels on the same stream: every sum must be of
    the written values (the consumers wait for the producer before their first input load).
    Narrow formats: the producer stores 64-bit words holding 2 (f32) / 4 (f16, bf16) copies of v."""
    import torch
    lib = synth.cuda_lib()
    st = torch.cuda.current_stream().cuda_stream
    for n, dt in ((1 << 20, torch.float64), (1 << 19, torch.float32), (1 << 21, torch.float16),
                  (1 << 21, torch.bfloat16), ((1 << 22) + 8, torch.float64)):
        y = torch.zeros(n, dtype=dt, device="cuda")
        words = y.view(torch.float64)
        per = 8 // y.element_size()
        acc = xs.Accumulator()
        for k in range(5):
            v = float(k + 1)
            word = float(torch.full((per,), v, dtype=dt).view(torch.float64).item())
            y.zero_()
            torch.cuda.synchronize()
            assert lib.synth_gpu_fill_after_trigger(words.data_ptr(), words.numel(), word, 200000, st) == 0
            res, _ = acc.sum(y)                      # launched right behind the producer
            got = xs.Result.from_bytes(res.cpu().numpy().tobytes()).value
            assert got == v * n, (n, dt, k, got)
