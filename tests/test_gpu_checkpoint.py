"""GPU tests of checkpoint / resume (the paper's external-memory scan keeps
the whole superaccumulator as the only state): a summation stopped after
any prefix, saved (xsum_save_state), resumed in a new accumulator (xsum_load_state) and
continued equals the oracle's exact sum of the whole input, bit for bit and in the canonical
image; corrupted checkpoints are rejected without touching the state."""
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


def dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def same(res, canon, r, limbs):
    return res.bits == r.bits and res.flags == r.flags and res.bits_f32 == r.bits_f32 and \
        (np.asarray(canon, dtype=np.uint64) == limbs).all()


@pytest.mark.parametrize("cfg,n,cuts", [("c2", 1 << 20, (0, 1, 777_777)), ("c3", 0, (123_457,)),
                                        ("c1", 100_003, (50_000, 50_001))])
def test_save_resume_continue(xs, tmp_path, cfg, n, cuts):
    x = synth.gen.generate(cfg, 0, n) if n else synth.gen.generate(cfg, 0, 1 << 18, permute=False)
    r, limbs = oracle.exact_sum(x)
    d = dev(x)
    acc = xs.Accumulator()
    prev = 0
    for k, c in enumerate(cuts):                      # stop, save, resume in a new accumulator
        acc.add(d[prev:c])
        path = tmp_path / f"ckpt{k}.xsum"
        acc.save(path)
        acc = xs.Accumulator.load(path)
        assert acc.count == c
        prev = c
    acc.add(d[prev:])
    assert acc.count == x.size
    res, canon = acc.exact()
    assert same(res, canon, r, limbs)


def test_resume_host_streaming_and_other_formats(xs):
    import torch
    x16 = synth.gen.bits("c2bf16", 0, 300_001)
    x = synth.gen.generate("c2", 5, 400_000)
    r, limbs = oracle.exact_sum(x)
    a = xs.Accumulator().add_host(torch.from_numpy(x[:123_456]).pin_memory(), stage_bytes=2 << 20)
    img = a.save_state()
    assert xs.check_state_image(img)
    b = xs.Accumulator().load_state(img).add_host(torch.from_numpy(x[123_456:]).pin_memory(), stage_bytes=2 << 20)
    res, canon = b.exact()
    assert same(res, canon, r, limbs)
    r16, l16 = oracle.exact_sum(x16, fmt="bf16")     # bfloat16 bit patterns, resumed mid-way
    t = dev(x16.view(np.int16)).view(torch.bfloat16)
    c = xs.Accumulator().add(t[:100_000])
    c2 = xs.Accumulator().load_state(c.save_state()).add(t[100_000:])
    res, canon = c2.exact()
    assert same(res, canon, r16, l16)


def test_flags_survive_checkpoint(xs):
    x = np.array([1.0, np.inf, 2.0, -np.inf, 3.0])
    a = xs.Accumulator().add(dev(x[:2]))
    b = xs.Accumulator().load_state(a.save_state()).add(dev(x[2:]))
    r, limbs = oracle.exact_sum(x)
    res, canon = b.exact()
    assert same(res, canon, r, limbs) and np.isnan(res.value)


def test_corrupted_checkpoint_rejected_state_kept(xs):
    x = synth.gen.generate("c2", 9, 50_000)
    a = xs.Accumulator().add(dev(x))
    good = a.save_state()
    r0 = a.result()
    for pos, val in ((0, 0x00), (6, 51), (24 + 8 * 5 + 6, 0x7F), (370, 1)):
        img = bytearray(good)
        img[pos] = val
        with pytest.raises(xs.XsumError) as e:
            a.load_state(bytes(img))
        assert e.value.status == 4                    # XSUM_EMISMATCH
    r1 = a.result()
    assert (r1.bits, r1.flags, r1.count) == (r0.bits, r0.flags, r0.count)
    with pytest.raises(ValueError):
        a.load_state(good[:100])
