"""Seeded input generators: the numpy definition (synth/gen.py), the threaded C
generator (synth/gen.c) and, on a GPU, the device generator (synth/csrc/gen.cu)
agree bit for bit; the generated workloads have the shapes BASELINE.json states."""
from __future__ import annotations

import numpy as np
import pytest

import synth
from synth import gen


def _exp(x: np.ndarray) -> np.ndarray:
    return ((x.view(np.uint64) >> np.uint64(52)) & np.uint64(0x7FF)).astype(np.int64) - 1023


def test_splitmix_reference_value():
    # splitmix64 of seed 0 (the first output of the classic generator state 0 + G)
    assert int(gen.mix64(np.array([0x9E3779B97F4A7C15], dtype=np.uint64))[0]) == 0xE220A8397B1DCDAF


@pytest.mark.parametrize("name,start", [("c1", 0), ("c2", 1 << 27), ("c4", (1 << 33) - 4096), ("c5", 77)])
def test_numpy_vs_c_uniform(name, start):
    a = gen.generate(name, start, 4096)
    b = synth.host_generate(name, start, 4096, nthreads=3)
    assert (a.view(np.uint64) == b.view(np.uint64)).all()


def test_numpy_vs_c_cancel():
    cfg = gen.CONFIGS["c3"]
    for start in (0, (1 << 28) - 1000, cfg["n"] - 1000):
        a = gen.generate("c3", start, 1000, permute=False)
        b = synth.host_generate("c3", start, 1000, nthreads=2)
        assert (a.view(np.uint64) == b.view(np.uint64)).all()
    k1 = gen.cancel_perm_keys(cfg, 5, 100)
    k2 = synth.host_keys(3, 2, 5, 100)
    assert (k1 == k2).all()


@pytest.mark.parametrize("name", ["c1", "c2", "c4", "c5"])
def test_uniform_shape(name):
    cfg = gen.CONFIGS[name]
    x = gen.generate(name, 0, 200_000)
    e = _exp(x)
    assert e.min() == cfg["lo"] and e.max() == cfg["hi"]          # inclusive exponent range
    assert np.isfinite(x).all()
    neg = (x < 0).mean()
    assert 0.49 < neg < 0.51                                       # random sign
    frac = x.view(np.uint64) & np.uint64((1 << 52) - 1)
    assert abs(float((frac >> np.uint64(51)).mean()) - 0.5) < 0.01  # uniform mantissa (top bit)
    counts = np.bincount(e - cfg["lo"])
    span = cfg["hi"] - cfg["lo"] + 1
    assert counts.size == span and counts.min() > 0.6 * x.size / span


def test_cancel_shape():
    cfg = gen.CONFIGS["c3"]
    x = gen.generate("c3", 0, 4000, permute=False)
    assert (x[0::2] == -x[1::2]).all()
    e = _exp(x)
    assert e.min() >= 0 and e.max() <= 600
    t = gen.generate("c3", 1 << 28, 4000, permute=False)
    et = _exp(t)
    assert et.min() >= -900 and et.max() <= -800
    assert cfg["n"] == (1 << 28) + (1 << 20)


def test_cancel_permutation_small_model():
    """The permutation is a stable sort of positions on their keys (checked on a prefix)."""
    cfg = dict(gen.CONFIGS["c3"])
    keys = gen.cancel_perm_keys(cfg, 0, 5000)
    perm = np.argsort(keys, kind="stable")
    assert sorted(perm.tolist()) == list(range(5000))
    assert (np.diff(keys[perm].astype(object)) >= 0).all()


@pytest.mark.gpu
@pytest.mark.parametrize("name,start", [("c1", 0), ("c2", 12345), ("c3", (1 << 28) - 100), ("c5", 1 << 20)])
def test_device_generator_matches_numpy(name, start):
    import torch
    synth.build()
    d = synth.device_generate(name, start, 10_000, permute=False)
    torch.cuda.synchronize()
    a = gen.generate(name, start, 10_000, permute=False)
    assert (d.cpu().numpy().view(np.uint64) == a.view(np.uint64)).all()


@pytest.mark.parametrize("name", ["c2f32", "c2f16", "c2bf16"])
def test_format_bits_numpy_vs_c(name):
    """The other-format workloads: numpy definition vs the threaded C draws, finite patterns only,
    every exponent field reached."""
    a = gen.bits(name, 1000, 200_000)
    b = synth.host_bits(name, 1000, 200_000)
    assert (a == b).all()
    width, em, _ = gen.FORMAT_BITS[gen.CONFIGS[name]["fmt"]]
    assert a.dtype == (np.uint32 if width == 32 else np.uint16)
    e = (a & a.dtype.type(em)) >> a.dtype.type((em & -em).bit_length() - 1)
    assert int(e.max()) == (em >> ((em & -em).bit_length() - 1)) - 1      # never all ones
    assert len(np.unique(e)) == int(e.max()) + 1                          # every finite exponent


def test_csr_workload_offsets():
    cfg = gen.CONFIGS["c5csr"]
    offs = gen.csr_offsets(cfg)
    lens = np.diff(offs)
    assert offs[0] == 0 and offs.size == cfg["nseg"] + 1 and offs[-1] == cfg["n"]
    assert lens.min() >= 1 and lens.max() <= cfg["maxlen"] and abs(lens.mean() - 4096) < 100


def test_f1_measurement_workloads():
    """c2dim0 is c2's element stream (viewed as [4096, 65536]); c5s16 draws like c5 with its own
    seed (exponents in [-200, 200], 2^24 segments of 16)."""
    import synth.gen as g
    a = g.generate("c2dim0", 12345, 1000)
    b = g.generate("c2", 12345, 1000)
    assert (a.view(np.uint64) == b.view(np.uint64)).all()
    assert g.CONFIGS["c2dim0"]["shape"][0] * g.CONFIGS["c2dim0"]["shape"][1] == g.CONFIGS["c2dim0"]["n"]
    c = g.CONFIGS["c5s16"]
    assert c["nseg"] * c["seg_len"] == c["n"]
    x = g.generate("c5s16", 0, 100_000)
    e = ((x.view(np.uint64) >> np.uint64(52)) & np.uint64(0x7FF)).astype(np.int64) - 1023
    assert e.min() >= -200 and e.max() <= 200 and e.min() < -190 and e.max() > 190
    assert not (x.view(np.uint64) == g.generate("c5", 0, 100_000).view(np.uint64)).all()
