"""GPU parity: the CUDA path (through the C-ABI) vs the oracle, bit for bit.

Every comparison checks the rounded double, the direction, the flags and the
canonical 34-limb image of the exact sum; integer work, so the
bar is bit-exactness (no tolerance). Inputs are seeded; expected values come only
from oracle/ (never from the CUDA path).
"""
from __future__ import annotations

import math
import random
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


def b2f(b: int) -> float:
    return struct.unpack("<d", struct.pack("<Q", b))[0]


def to_dev(x: np.ndarray, offset: int = 0):
    """Copy to the GPU; offset=1 gives a base that is 8-B but not 16-B aligned."""
    import torch
    buf = torch.empty(x.size + 2, dtype=torch.float64, device="cuda")
    assert buf.data_ptr() % 16 == 0
    t = buf[offset:offset + x.size]
    t.copy_(torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)))
    return t


def assert_same(res, canon, x: np.ndarray | None = None, ref=None, what: str = ""):
    if ref is None:
        ref = oracle.exact_sum(x)
    r, limbs = ref
    assert res.bits == r.bits, f"{what}: value {res.bits:016x} != oracle {r.bits:016x}"
    assert res.direction == r.direction, what
    assert res.flags == r.flags, f"{what}: flags {res.flags} != {r.flags}"
    assert res.msb_exp == r.msb_exp and res.sign == r.sign, what
    assert res.sig53 == r.sig53 and res.exp2 == r.exp2, what
    assert res.bits_f32 == r.bits_f32, f"{what}: binary32 {res.bits_f32:08x} != oracle {r.bits_f32:08x}"
    if canon is not None:
        assert (np.asarray(canon, dtype=np.uint64) == limbs).all(), f"{what}: canonical image differs"


# ---------------------------------------------------------------------------------------
# edge cases and small random sets
# ---------------------------------------------------------------------------------------

def test_golden_cases(xs):
    from test_oracle_pins import GOLDEN_CASES
    for name, xs_, out_bits, direction, _ in GOLDEN_CASES:
        x = np.array(xs_, dtype=np.float64)
        for off in (0, 1):
            res, canon = xs.exact_sum(to_dev(x, off))
            assert res.bits == out_bits, name
            assert res.direction == direction, name
            assert_same(res, canon, x, what=name)


def _rand_set(rng: random.Random, n: int) -> list[float]:
    from test_oracle_pins import _random_set
    xs_ = _random_set(rng, n)
    if rng.random() < 0.05 and xs_:   # a few specials
        xs_[rng.randrange(len(xs_))] = rng.choice([math.inf, -math.inf, math.nan, b2f(0x7FF0000000000001)])
    return xs_


def test_many_small_sets_via_csr_segments(xs):
    import torch
    rng = random.Random(2024)
    sets = [_rand_set(rng, rng.choice([0, 1, 2, 3, 5, 8, 13, 31, 32, 33, 64, 65, 200, 257, 1000]))
            for _ in range(3000)]
    offs = np.cumsum([0] + [len(s) for s in sets]).astype(np.int64)
    flat = np.array([v for s in sets for v in s], dtype=np.float64)
    vals, canon, flags = xs.sum_segments_csr(to_dev(flat), torch.from_numpy(offs).cuda(), canon=True, flags=True)
    vals = vals.cpu().numpy().view(np.uint64)
    canon = canon.cpu().numpy().view(np.uint64)
    flags = flags.cpu().numpy()
    for k, s in enumerate(sets):
        r, limbs = oracle.exact_sum(np.array(s, dtype=np.float64))
        assert int(vals[k]) == r.bits, (k, s)
        assert int(flags[k]) == r.flags, k
        assert (canon[k] == limbs).all(), k


@pytest.mark.parametrize("n", [0, 1, 2, 3, 31, 32, 33, 63, 64, 65, 1023, 1024, 1025, 4095, 4096, 4097,
                               8191, 8192, 8193, 65535, 65537, 148 * 4096 - 1, 148 * 4096 + 3,
                               1016 * 512 * 2 + 7, 5_000_017])
@pytest.mark.parametrize("off", [0, 1])
def test_sizes_alignment_both_paths(xs, n, off):
    x = synth.gen.generate("c4", 77, n) if n else np.zeros(0)
    d = to_dev(x, off)
    ref = oracle.exact_sum(x)
    res, canon = xs.exact_sum(d)                       # fused one-launch path (xsum_sum)
    assert_same(res, canon, ref=ref, what=f"fused n={n} off={off}")
    acc = xs.Accumulator()                             # create / accumulate / finalize path
    acc.add(d)
    res2, canon2 = acc.exact()
    assert_same(res2, canon2, ref=ref, what=f"acc n={n} off={off}")
    assert res2.count == n


@pytest.mark.parametrize("blocks", [1, 2, 3, 7])
def test_many_flush_windows_per_lane(xs, blocks):
    """A capped grid forces each lane through many regularization windows (FLUSH_ELEMS),
    with NaN/Inf patterns planted across windows (rescan path) and a ragged tail."""
    n = 3 * 1016 * 512 * 2 * blocks + 4097 * blocks + 5
    x = synth.gen.generate("c4", 999, n)
    ref_finite = oracle.exact_sum(x)
    acc = xs.Accumulator().set_grid_limit(blocks)
    for off in (0, 1):
        res, canon = acc.sum(to_dev(x, off), canon=True)
        assert_same(xs.Result.from_bytes(res.cpu().numpy().tobytes()), canon.cpu().numpy().view(np.uint64),
                    ref=ref_finite, what=f"blocks={blocks} off={off}")
    y = x.copy()
    rng = np.random.default_rng(blocks)
    for i in rng.choice(n, size=40, replace=False):
        y.view(np.uint64)[i] = rng.choice([0x7FF0000000000000, 0xFFF0000000000000, 0x7FF8000000000001])
    acc.reset().add(to_dev(y))
    res, canon = acc.exact()
    assert_same(res, canon, y, what=f"specials blocks={blocks}")


@pytest.mark.parametrize("sign", [1.0, -1.0, 0.0])
def test_headroom_worst_case_digits(xs, sign):
    """Every summand produces the largest chunks (M = 2^53-1 at offset o = 51 in its digit),
    all lanes hit the same digit, each lane takes full flush windows plus stragglers: the
    raw lane digits reach the int64 headroom bound the kernel's schedule relies on
    (xsum_device.cuh FLUSH_ELEMS) and the raw-column combine sees its largest inputs."""
    import math
    v = math.ldexp((1 << 53) - 1, 17)                  # e = 1092: k = 1091 = 52*20 + 51
    n = 512 * 2032 * 3 + 4099
    x = np.full(n, v if sign >= 0 else -v)
    if sign == 0.0:                                    # alternate signs in runs
        x[(np.arange(n) // 7) % 2 == 1] *= -1
    acc = xs.Accumulator().set_grid_limit(1)
    for off in (0, 1):
        res, canon = acc.sum(to_dev(x, off), canon=True)
        assert_same(xs.Result.from_bytes(res.cpu().numpy().tobytes()), canon.cpu().numpy().view(np.uint64),
                    x, what=f"headroom sign={sign} off={off}")
    vals, canon2, _ = xs.sum_segments(to_dev(x[: 256 * 2100 * 2]), 256 * 2100, canon=True)
    for s in range(2):
        r, limbs = oracle.exact_sum(x[s * 256 * 2100:(s + 1) * 256 * 2100])
        assert int(vals.cpu().numpy().view(np.uint64)[s]) == r.bits
        assert (canon2.cpu().numpy().view(np.uint64)[s] == limbs).all()


def test_chunked_accumulate_random_splits(xs):
    rng = np.random.default_rng(5)
    x = synth.gen.generate("c2", 0, 3_000_000)
    d = to_dev(x)
    ref = oracle.exact_sum(x)
    for trial in range(5):
        cuts = np.sort(rng.integers(0, x.size, size=rng.integers(1, 12)))
        cuts = [0, *cuts.tolist(), x.size]
        acc = xs.Accumulator()
        for a, b in zip(cuts, cuts[1:]):
            acc.add(d[a:b])
        res, canon = acc.exact()
        assert_same(res, canon, ref=ref, what=f"split {cuts}")


def test_host_buffer_path(xs):
    import torch
    x = synth.gen.generate("c4", 1 << 30, 5_000_001)
    ref = oracle.exact_sum(x)
    pinned = torch.from_numpy(x).pin_memory()
    acc = xs.Accumulator()
    acc.add_host(pinned, stage_bytes=4 << 20)          # many double-buffered chunks
    res, canon = acc.exact()
    assert_same(res, canon, ref=ref, what="host path")
    acc2 = xs.Accumulator().add_host(x)                # pageable numpy buffer
    res2, canon2 = acc2.exact()
    assert_same(res2, canon2, ref=ref, what="host path pageable")


def test_permutation_invariance(xs):
    rng = np.random.default_rng(9)
    x = synth.gen.generate("c2", 10, 2_000_000)
    base = xs.exact_sum(to_dev(x))
    for _ in range(3):
        res, canon = xs.exact_sum(to_dev(rng.permutation(x)))
        assert res.bits == base[0].bits and (canon == base[1]).all()
    assert_same(base[0], base[1], x)


def test_specials_in_hot_loop_and_tails(xs):
    """NaN/Inf patterns anywhere (main tiles, leftovers, head, tail) are flagged and do
    not perturb the exact finite part (the rare rescan path of accumulate.cu)."""
    rng = np.random.default_rng(1)
    n = 4 * 1016 * 512 * 2 + 999
    base = synth.gen.generate("c2", 0, n)
    cases = {
        "nan_mid": [(n // 3, 0x7FF8000000000000)],
        "pinf_head": [(0, 0x7FF0000000000000)],
        "ninf_tail": [(n - 1, 0xFFF0000000000000)],
        "snan_payload": [(12345, 0x7FF0000000000001), (n - 700, 0x7FF0000000000002)],
        "both_inf": [(5, 0x7FF0000000000000), (n // 2, 0xFFF0000000000000)],
        "many": [(int(i), 0x7FF0000000000000 | int(rng.integers(0, 2)) << 63) for i in
                 rng.choice(n, size=5000, replace=False)],
    }
    for name, plants in cases.items():
        x = base.copy()
        xb = x.view(np.uint64)
        for i, bits in plants:
            xb[i] = bits
        for off in (0, 1):
            res, canon = xs.exact_sum(to_dev(x, off))
            assert_same(res, canon, x, what=f"{name} off={off}")


# ---------------------------------------------------------------------------------------
# merge (MapReduce post-process / all-gather path) and Lemma-1 stress
# ---------------------------------------------------------------------------------------

def test_merge_of_shard_states_equals_whole(xs):
    import torch
    from paper_1605_05436_b200 import dist
    x = synth.gen.generate("c4", 0, 4_000_003)
    d = to_dev(x)
    ref = oracle.exact_sum(x)
    for p in (1, 2, 3, 8, 37):
        states = []
        for r in range(p):
            a, b = dist.shard_range(x.size, r, p)
            states.append(xs.Accumulator().add(d[a:b]).state.clone())
        blob = torch.cat(states[::-1])                 # any order
        acc = xs.Accumulator().merge(blob)
        res, canon = acc.exact()
        assert_same(res, canon, ref=ref, what=f"merge p={p}")
        assert res.count == x.size


def test_merge_round_is_the_fused_post_process(xs):
    """xsum_merge_round: state := sum of the images (previous state discarded), rounded in the
    same launch - the multi-GPU step's post-process after the all-gather."""
    import torch
    from paper_1605_05436_b200 import dist
    x = synth.gen.generate("c4", 1 << 32, 3_000_017)
    d = to_dev(x)
    ref = oracle.exact_sum(x)
    states = []
    for r in range(8):
        a, b = dist.shard_range(x.size, r, 8)
        acc = xs.Accumulator()
        acc.sum(d[a:b])                              # the local fused step each rank runs
        states.append(acc.state.clone())
    tot = xs.Accumulator().add(d[:1000])             # stale content must be discarded
    n0 = xs.launch_count()
    res, canon = tot.merge_round(torch.cat(states), canon=True)
    assert xs.launch_count() - n0 == 1
    assert_same(xs.Result.from_bytes(res.cpu().numpy().tobytes()), canon.cpu().numpy().view(np.uint64),
                ref=ref, what="merge_round")
    r2, c2 = tot.exact()                             # the state holds the merged sum
    assert_same(r2, c2, ref=ref, what="merge_round state")


def _image(digits, count=0, flags=0, magic=0x4D555358):
    from test_host_logic import encode_state
    img = encode_state(0, count, flags)
    img[0:4] = np.array([magic], dtype=np.uint32).view(np.uint8)
    img[24:24 + 8 * 42] = np.array(digits, dtype=np.int64).view(np.uint8)
    return img


def test_lemma1_merge_adversarial_digits(xs):
    """Regularized digits at the Lemma-1 boundaries (P_j = +-(R-1), +-(2R-2)) merged in a
    tree; the canonical image must equal the exact integer sum of the digit vectors."""
    import torch
    R = 1 << 52
    rng = random.Random(4)
    pats = []
    for _ in range(64):
        kind = rng.random()
        if kind < 0.3:
            d = [rng.choice([R - 1, -(R - 1)]) for _ in range(41)]
        elif kind < 0.6:
            d = [rng.choice([R - 1, -(R - 1), 0, 1, -1, R // 2, -(R // 2)]) for _ in range(41)]
        else:
            d = [rng.randint(-(R - 1), R - 1) for _ in range(41)]
        d.append(rng.randint(-(1 << 20), 1 << 20))
        pats.append(d)
    for k in (1, 2, 5, 16, 17, 64):
        imgs = np.concatenate([_image(p) for p in pats[:k]])
        acc = xs.Accumulator().merge(torch.from_numpy(imgs).cuda())
        res, canon = acc.exact()
        A = sum(sum(v << (52 * j) for j, v in enumerate(p)) for p in pats[:k])
        ref_r = oracle.round_limbs(oracle.int_to_limbs(A), 0, 0)
        assert (canon == oracle.int_to_limbs(A)).all(), k
        assert res.bits == ref_r.bits and res.direction == ref_r.direction, k
        assert res.flags == ref_r.flags


def test_merge_rejects_bad_images(xs):
    import torch
    good = _image([1] + [0] * 41, count=3)
    bad_magic = _image([5] + [0] * 41, magic=0x12345678)
    bad_digit = _image([1 << 52] + [0] * 41)          # not regularized (|Y| > R-1)
    acc = xs.Accumulator().merge(torch.from_numpy(np.concatenate([good, bad_magic, bad_digit])).cuda())
    res, canon = acc.exact()
    assert res.flags & xs.F_MISMATCH
    assert res.bits == 1 and res.count == 3            # only the good image counted: 2^-1074


@pytest.mark.parametrize("k", [17, 40, 100])
def test_merge_rejects_bad_images_past_first_leaf_round(xs, k):
    """k images through the 16 leaf warps' pipelined loads (image s + 16 in flight while s folds):
    malformed images at positions 16, 20, 33 and 99 (when present) are rejected, the rest counted."""
    import torch
    imgs, good_count = [], 0
    for i in range(k):
        if i in (16, 33):
            imgs.append(_image([5] + [0] * 41, magic=0x12345678))
        elif i in (20, 99):
            imgs.append(_image([1 << 52] + [0] * 41))
        else:
            imgs.append(_image([1] + [0] * 41, count=3))
            good_count += 1
    res, canon = xs.Accumulator().merge(torch.from_numpy(np.concatenate(imgs)).cuda()).exact()
    assert res.flags & xs.F_MISMATCH
    assert res.bits == good_count and res.count == 3 * good_count       # good_count * 2^-1074


def test_launch_counter_counts_kernels(xs):
    n0 = xs.launch_count()
    acc = xs.Accumulator()              # init kernel
    acc.add(to_dev(np.ones(1000)))      # one accumulate kernel
    acc.result()                        # one finalize kernel
    assert xs.launch_count() - n0 == 3


# ---------------------------------------------------------------------------------------
# segmented sums (config 5 and ragged)
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("seg_len,off", [(1, 1), (2, 1), (3, 0), (31, 1), (33, 0), (127, 1), (4096, 1), (5000, 0),
                                         (1016 * 64 + 3, 1), (256, 0), (512, 0), (4096, 0), (256 * 300, 0)])
def test_segments_ragged_lengths(xs, seg_len, off):
    """Equal segments: misaligned / ragged lengths take the general kernel, aligned multiples
    of 256 the streaming fast path (incl. a segment longer than one flush window). NaN/Inf
    patterns planted in the first and the last segment."""
    nseg = max(1, min(300, 2_000_000 // seg_len))
    x = synth.gen.generate("c5", 3, nseg * seg_len)
    xb = x.view(np.uint64)
    xb[7 % x.size] = 0x7FF8000000000000                        # NaN in segment 0
    xb[x.size - 1 - (5 % seg_len)] = 0xFFF0000000000000        # -Inf in the last segment
    if seg_len > 70000:
        xb[seg_len // 2 + 3] = 0x7FF0000000000000              # +Inf in a later flush window
    vals, canon, flags = xs.sum_segments(to_dev(x, off), seg_len, canon=True, flags=True)
    vals = vals.cpu().numpy().view(np.uint64)
    canon = canon.cpu().numpy().view(np.uint64)
    flags = flags.cpu().numpy()
    for s in range(nseg):
        r, limbs = oracle.exact_sum(x[s * seg_len:(s + 1) * seg_len])
        assert int(vals[s]) == r.bits and int(flags[s]) == r.flags and (canon[s] == limbs).all(), s


# ---------------------------------------------------------------------------------------
# full BASELINE.json configs (c1..c5), inputs from the device generator; expected values
# from the oracle over the host generator's identical bytes
# ---------------------------------------------------------------------------------------

def _host_config(name: str) -> np.ndarray:
    return synth.host_generate(name)            # c3: pre-permutation order (sum is order-free)


def _check_device_input_sample(name: str, d):
    """The device generator produced the same bytes as the host generator (sampled)."""
    if name == "c3":
        return
    n = d.numel()
    for start in (0, n // 2, n - 4096):
        a = synth.gen.generate(name, start, 4096)
        assert (d[start:start + 4096].cpu().numpy().view(np.uint64) == a.view(np.uint64)).all()


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_full_config_parity(xs, name):
    import torch
    d = synth.device_generate(name)
    _check_device_input_sample(name, d)
    res, canon = xs.exact_sum(d)
    del d
    torch.cuda.empty_cache()
    ref = oracle.exact_sum(_host_config(name))
    assert_same(res, canon, ref=ref, what=name)
    if name == "c3":   # the exact sum is the sum of the tiny terms alone
        cfg = synth.CONFIGS["c3"]
        tiny = synth.gen.generate("c3", 2 * cfg["npairs"], cfg["ntiny"], permute=False)
        r_t, l_t = oracle.exact_sum(tiny)
        assert (l_t == canon).all() and r_t.bits == res.bits


def test_full_config_c5_segments(xs):
    d = synth.device_generate("c5")
    cfg = synth.CONFIGS["c5"]
    vals, canon, flags = xs.sum_segments(d, cfg["seg_len"], canon=True, flags=True)
    vals = vals.cpu().numpy().view(np.uint64)
    canon = canon.cpu().numpy().view(np.uint64)
    flags = flags.cpu().numpy()
    host = _host_config("c5")
    L = cfg["seg_len"]
    for s in range(cfg["nseg"]):
        r, limbs = oracle.exact_sum(host[s * L:(s + 1) * L], nthreads=1)
        assert int(vals[s]) == r.bits and int(flags[s]) == r.flags and (canon[s] == limbs).all(), s


@pytest.mark.slow
def test_full_config_c4_one_gpu(xs):
    """n = 2^33 (64 GiB) on one GPU, fused path (the bench's launch configuration);
    the oracle streams the same 2^33 doubles from the host generator in chunks."""
    import torch
    free, _ = torch.cuda.mem_get_info()
    cfg = synth.CONFIGS["c4"]
    if free < cfg["n"] * 8 + (4 << 30):
        pytest.skip("not enough device memory for 64 GiB")
    d = synth.device_generate("c4")
    res, canon = xs.exact_sum(d)
    del d
    torch.cuda.empty_cache()
    acc = oracle.Accumulator()
    chunk = 1 << 26
    buf = np.empty(chunk, dtype=np.float64)
    for start in range(0, cfg["n"], chunk):
        acc.add(synth.host_generate("c4", start, chunk, out=buf))
    assert_same(res, canon, ref=(acc.result(), acc.limbs), what="c4")
    assert math.isinf(res.value) or res.msb_exp < 1024      # (Q12: almost surely +-Inf)


# ---------------------------------------------------------------------------------------
# binary32 inputs
# ---------------------------------------------------------------------------------------

def _f32_data(n: int, seed: int, emin: int = 1, emax: int = 254) -> np.ndarray:
    rng = np.random.default_rng(seed)
    e = rng.integers(emin, emax + 1, size=n, dtype=np.uint32)
    bits = (rng.integers(0, 2, size=n, dtype=np.uint32) << np.uint32(31)) | (e << np.uint32(23)) | \
        rng.integers(0, 1 << 23, size=n, dtype=np.uint32)
    return bits.view(np.float32)


def to_dev32(x: np.ndarray, offset: int = 0):
    import torch
    buf = torch.empty(x.size + 4, dtype=torch.float32, device="cuda")
    t = buf[offset:offset + x.size]
    t.copy_(torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)))
    return t


@pytest.mark.parametrize("n", [0, 1, 3, 4, 5, 17, 4095, 4096 * 4 + 3, 65536 + 7, 148 * 8192 + 11, 3_000_001])
@pytest.mark.parametrize("off", [0, 1, 2, 3])
def test_f32_sizes_alignment(xs, n, off):
    x = _f32_data(n, n + 17 * off)
    if n > 10:                                   # subnormals and zeros too
        x[::97] = np.float32(1e-42)
        x[5::101] = np.float32(-0.0)
    ref = oracle.exact_sum(x)
    d = to_dev32(x, off)
    res, canon = xs.exact_sum(d)
    assert_same(res, canon, ref=ref, what=f"f32 fused n={n} off={off}")
    acc = xs.Accumulator().add(d)
    res2, canon2 = acc.exact()
    assert_same(res2, canon2, ref=ref, what=f"f32 acc n={n} off={off}")


@pytest.mark.parametrize("blocks", [1, 3])
def test_f32_flush_windows_and_specials(xs, blocks):
    n = 3 * 2016 * 512 * blocks + 777
    x = _f32_data(n, blocks, 100, 160)
    acc = xs.Accumulator().set_grid_limit(blocks)
    res, canon = acc.sum(to_dev32(x), canon=True)
    assert_same(xs.Result.from_bytes(res.cpu().numpy().tobytes()), canon.cpu().numpy().view(np.uint64),
                x, what=f"f32 windows blocks={blocks}")
    y = x.copy()
    rng = np.random.default_rng(7)
    for i in rng.choice(n, size=25, replace=False):
        y.view(np.uint32)[i] = rng.choice([0x7F800000, 0xFF800000, 0x7FC00001])
    acc.reset().add(to_dev32(y, 1))
    res, canon = acc.exact()
    assert_same(res, canon, y, what=f"f32 specials blocks={blocks}")


def test_f32_signed_zeros_and_subnormals(xs):
    """-0.0f has M = 0 with the sign bit set; subnormals have no hidden bit (R2)."""
    rng = np.random.default_rng(4)
    subs = (rng.integers(1, 1 << 23, size=9000, dtype=np.uint32) |
            (rng.integers(0, 2, size=9000, dtype=np.uint32) << np.uint32(31))).view(np.float32)
    for x in (np.array([-0.0], np.float32), np.array([-0.0, 0.0, -0.0], np.float32),
              np.full(70000, -0.0, np.float32), subs, np.concatenate([subs, np.full(555, -0.0, np.float32)])):
        res, canon = xs.exact_sum(to_dev32(x, 1))
        assert_same(res, canon, x, what=f"f32 zeros/subnormals n={x.size}")


def test_mixed_binary32_and_binary64_in_one_state(xs):
    """One superaccumulator holds binary32 and binary64 summands exactly (same 2^-1074 window)."""
    a = _f32_data(1_000_003, 3, 60, 200)
    b = synth.gen.generate("c2", 0, 2_000_001)
    acc = xs.Accumulator().add(to_dev32(a)).add(to_dev(b, 1)).add(to_dev32(-a[:1000]))
    res, canon = acc.exact()
    oa = oracle.Accumulator().add(a).add(b).add(-a[:1000])
    assert_same(res, canon, ref=(oa.result(), oa.limbs), what="mixed")


def test_status_codes_on_device(xs):
    """Argument errors are reported as status codes (never crashes), on a live device."""
    import ctypes

    import torch
    L = xs.lib()
    acc = xs.Accumulator()
    d = torch.zeros(16, dtype=torch.float64, device="cuda")
    f = torch.zeros(16, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    assert L.xsum_accumulate(acc.handle, d.data_ptr() + 4, 3, st) == xs.EINVAL       # not 8-B aligned
    assert L.xsum_accumulate_f32(acc.handle, f.data_ptr() + 2, 3, st) == xs.EINVAL   # not 4-B aligned
    assert L.xsum_accumulate(acc.handle, None, 3, st) == xs.EINVAL
    assert L.xsum_accumulate(acc.handle, d.data_ptr(), 0, st) == xs.OK               # n = 0: no-op
    assert L.xsum_merge(acc.handle, d.data_ptr() + 4, 1, st) == xs.EINVAL
    assert L.xsum_finalize_round(acc.handle, None, None, st) == xs.EINVAL
    assert L.xsum_accumulate(acc.handle, d.data_ptr(), 2 ** 63, st) == xs.ECAPACITY   # > 2^63-1 summands
    h = ctypes.c_void_p()
    small = torch.zeros(16, dtype=torch.uint8, device="cuda")
    assert L.xsum_create(ctypes.byref(h), 0, acc.state.data_ptr(), small.data_ptr(), 16, st) == xs.EINVAL
    assert L.xsum_create(ctypes.byref(h), 99, acc.state.data_ptr(), acc.scratch.data_ptr(),
                         acc.scratch.numel(), st) == xs.EINVAL
    with pytest.raises((TypeError, xs.XsumError)):
        acc.merge(torch.zeros(100, dtype=torch.uint8, device="cuda"))             # not k*384 bytes
    torch.cuda.synchronize()
    assert acc.result().count == 0 and acc.result().bits == 0                    # state untouched


def test_many_state_images_merge(xs):
    """A merge of thousands of states (the Lemma-1 leaf folds plus the warp tree)."""
    import torch
    x = synth.gen.generate("c4", 77, 2_000_000)
    d = to_dev(x)
    k = 2500
    cuts = np.linspace(0, x.size, k + 1).astype(int)
    states = torch.empty((k, 384), dtype=torch.uint8, device="cuda")
    acc = xs.Accumulator()
    for j in range(k):
        acc.sum(d[cuts[j]:cuts[j + 1]])
        states[j].copy_(acc.state)
    res, canon = xs.Accumulator().merge(states.reshape(-1)).exact()
    assert_same(res, canon, x, what="2500-way merge")
    assert res.count == x.size


@pytest.mark.parametrize("shape,dim", [((7, 300), -1), ((7, 300), 0), ((3, 5, 4097), 1), ((2, 0, 3), 2),
                                       ((2, 0, 3), 1), ((1,), 0), ((4, 1), 1), ((33, 2049), 0)])
def test_exact_sum_dim(xs, shape, dim):
    """Exact reduction along a tensor dimension: each fibre vs the oracle."""
    import torch
    n = int(np.prod(shape))
    x = synth.gen.generate("c2", 11, n).reshape(shape) if n else np.zeros(shape)
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    out = xs.exact_sum_dim(t, dim).cpu().numpy()
    ref_shape = np.sum(x, axis=dim).shape
    assert out.shape == ref_shape
    xm = np.moveaxis(x, dim, -1).reshape(out.size, x.shape[dim])
    for i, row in enumerate(xm):
        r, _ = oracle.exact_sum(row)
        assert out.reshape(-1)[i].view(np.uint64) == np.uint64(r.bits), (shape, dim, i)
    kd = xs.exact_sum_dim(t, dim, keepdim=True)
    assert tuple(kd.shape) == tuple(np.sum(x, axis=dim, keepdims=True).shape)


def test_every_exponent_and_digit_boundary(xs):
    """Per-element decomposition at every binary64 exponent (SURVEY.md §4 layer 3): each
    biased exponent 0..2046 with a random fraction and both signs, summed alone (segments of
    length 1) and with its neighbour one exponent up (the chunks straddle every digit boundary
    k mod 52 = 0 and 51), each vs the oracle."""
    import torch
    rng = np.random.default_rng(2046)
    e = np.arange(2047, dtype=np.uint64)
    frac = rng.integers(0, 1 << 52, size=e.size, dtype=np.uint64)
    sign = rng.integers(0, 2, size=e.size, dtype=np.uint64)
    bits = (sign << np.uint64(63)) | (e << np.uint64(52)) | frac
    x = bits.view(np.float64)
    d = torch.from_numpy(x.copy()).cuda()
    vals, canon, flags = xs.sum_segments(d, 1, canon=True, flags=True)
    v, cn = vals.cpu().numpy().view(np.uint64), canon.cpu().numpy().view(np.uint64)
    for i in range(x.size):
        r, limbs = oracle.exact_sum(x[i:i + 1])
        assert v[i] == r.bits and (cn[i] == limbs).all(), f"exponent field {i}"
    pairs = np.stack([x[:-1], -x[1:] * 0.75], axis=1).reshape(-1)
    vals, canon, _ = xs.sum_segments(torch.from_numpy(pairs.copy()).cuda(), 2, canon=True)
    v, cn = vals.cpu().numpy().view(np.uint64), canon.cpu().numpy().view(np.uint64)
    for i in range(x.size - 1):
        r, limbs = oracle.exact_sum(pairs[2 * i:2 * i + 2])
        assert v[i] == r.bits and (cn[i] == limbs).all(), f"pair at exponent field {i}"
    res, canon = xs.exact_sum(d)                          # and all of them at once (fused path)
    r, limbs = oracle.exact_sum(x)
    assert res.bits == r.bits and (canon == limbs).all()


@pytest.mark.parametrize("seg_len,nseg", [(512, 1), (512, 301), (1024, 77), (8192, 5), (4096, 2049)])
def test_segments_half_warp_path(xs, seg_len, nseg):
    """K6h (half a warp per segment, equal 16-B-aligned segments of a multiple of 512): odd
    segment counts (the last pair's second half idles and writes nothing), NaN / Inf planted in
    the last segment and in a segment the other half of its warp does not see, canonical images
    and flags of every segment vs the oracle."""
    x = synth.gen.generate("c5", 11, nseg * seg_len)
    xb = x.view(np.uint64)
    xb[x.size - 3] = 0x7FF0000000000000                        # +Inf in the last segment
    if nseg > 2:
        xb[seg_len + 5] = 0x7FF8000000000001                   # NaN in segment 1
        xb[2 * seg_len + 9] = 0xFFF0000000000000               # -Inf in segment 2
    vals, canon, flags = xs.sum_segments(to_dev(x, 0), seg_len, canon=True, flags=True)
    vals = vals.cpu().numpy().view(np.uint64)
    canon = canon.cpu().numpy().view(np.uint64)
    flags = flags.cpu().numpy()
    for s in range(nseg):
        r, limbs = oracle.exact_sum(x[s * seg_len:(s + 1) * seg_len], nthreads=1)
        assert int(vals[s]) == r.bits and int(flags[s]) == r.flags and (canon[s] == limbs).all(), s


def _band_segments(rng, nseg: int, seg_len: int) -> np.ndarray:
    """Segments whose exponent bands differ (K6z combines only the digits a half-warp's segment
    touched, positions relative to the band's lowest digit): narrow bands anywhere in the range,
    bands straddling the 16-digit row groups, the full range, cancellation to a tiny or subnormal
    sum, zeros and subnormal inputs (band from digit 0), specials, exact ties, overflow."""
    out = np.empty((nseg, seg_len), dtype=np.uint64)

    def field(lo, hi, n):
        e = rng.integers(max(lo, 0), min(hi, 2046) + 1, n, dtype=np.uint64)
        m = rng.integers(0, 1 << 52, n, dtype=np.uint64)
        s = rng.integers(0, 2, n, dtype=np.uint64)
        return (s << np.uint64(63)) | (e << np.uint64(52)) | m

    for s in range(nseg):
        kind = s % 11
        if kind == 0:
            c = int(rng.integers(1, 2047))
            v = field(c - 30, c + 30, seg_len)
        elif kind == 1:
            v = field(1, 2046, seg_len)
        elif kind == 2:                                 # pairs a, -a and a few tiny terms
            h = field(600, 1400, seg_len // 2)
            v = np.concatenate([h, h ^ np.uint64(1 << 63)])
            v[:4] = field(1, 40, 4)
            rng.shuffle(v)
        elif kind == 3:                                 # zeros, subnormals and normals
            v = field(900, 1100, seg_len)
            idx = rng.integers(0, seg_len, seg_len // 8)
            v[idx] = rng.integers(0, 1 << 52, idx.size, dtype=np.uint64)            # subnormal / zero
            v[idx[: idx.size // 2]] = np.uint64(0)
        elif kind == 4:                                 # a special
            v = field(500, 700, seg_len)
            v[int(rng.integers(0, seg_len))] = rng.choice(np.array([0x7FF0000000000000, 0xFFF0000000000000,
                                                                    0x7FF8000000000123], dtype=np.uint64))
        elif kind == 5:                                 # all (signed) zeros
            v = (rng.integers(0, 2, seg_len, dtype=np.uint64) << np.uint64(63))
        elif kind == 6:                                 # an exact tie: 2^53 + 1 (+ even/odd neighbours)
            v = np.zeros(seg_len, dtype=np.uint64)
            v[0] = np.float64(2.0 ** 53).view(np.uint64)
            v[seg_len // 2] = np.float64(1.0).view(np.uint64)
            v[seg_len - 1] = np.float64(2.0 * (s % 2)).view(np.uint64)
        elif kind == 7:                                 # around the digit-16 row boundary (k ~ 832)
            v = field(800, 870, seg_len)
        elif kind == 8:                                 # around the digit-32 row boundary (k ~ 1664)
            v = field(1630, 1700, seg_len)
        elif kind == 9:                                 # overflow of the rounded sum
            v = field(2046, 2046, seg_len) & np.uint64((1 << 63) - 1)
        else:                                           # cancellation to a subnormal sum
            h = field(1, 3, seg_len // 2)
            v = np.concatenate([h, h ^ np.uint64(1 << 63)])
            v[0] = np.uint64(5)
            rng.shuffle(v)
        out[s] = v
    return out.reshape(-1).view(np.float64)


@pytest.mark.parametrize("seg_len,nseg", [(512, 45), (768, 21), (1024, 23), (1280, 15), (4096, 33), (8192, 11), (15872, 11),
                                         (16128, 3), (16384, 5)])
def test_segments_half_band_values_only(xs, seg_len, nseg):
    """Values-only equal segments (K6z's banded epilogue: no canonical image requested) with a
    different exponent band in every segment and both halves of a warp on different bands: value
    and flags of every segment vs the oracle; 16384 (1024 summands per lane) takes K6h."""
    rng = np.random.default_rng(1605 + seg_len)
    x = _band_segments(rng, nseg, seg_len)
    vals, _, flags = xs.sum_segments(to_dev(x, 0), seg_len, flags=True)
    vals = vals.cpu().numpy().view(np.uint64)
    flags = flags.cpu().numpy()
    for s in range(nseg):
        r, _ = oracle.exact_sum(x[s * seg_len:(s + 1) * seg_len], nthreads=1)
        assert int(vals[s]) == r.bits and int(flags[s]) == r.flags, (s, s % 11, hex(int(vals[s])), hex(r.bits))
    # the same segments with images requested (the full-width epilogue) agree as well
    vals2, canon, _ = xs.sum_segments(to_dev(x, 0), seg_len, canon=True)
    assert (vals2.cpu().numpy().view(np.uint64) == vals).all()


@pytest.mark.parametrize("fill", ["pairs", "zeros"])
def test_segments_half_fast_rounding_boundaries(xs, fill):
    """K6z's banded rounding at its boundaries: segments of 512 whose sum is a binary64 / binary32
    tie or an ulp from a rounding boundary in the top digits, tipped either way (or not) by tiny
    terms several digits lower, both signs, exponents over the whole range; the rest of each
    segment cancelling pairs near the top (a narrow band: one row group) or zeros (the band starts
    at digit 0: three row groups). Values and flags (both roundings) vs the oracle."""
    import torch
    rng = np.random.default_rng(811 if fill == "pairs" else 812)
    nseg, L = 2048, 512
    x = np.zeros((nseg, L))
    for s in range(nseg):
        e = int(rng.integers(-900, 960))
        sg = 1.0 if rng.random() < 0.5 else -1.0
        prec = 53 if rng.random() < 0.5 else 24
        m = float(rng.integers(1 << 20, 1 << 21))
        top = sg * m * 2.0 ** e
        half = 2.0 ** (e + 20 - prec) * (1 if rng.random() < 0.7 else 2)
        x[s, 0] = top
        x[s, 1] = sg * half * (1 if rng.random() < 0.8 else -1)
        tiny_e = e - int(rng.integers(60, 300))
        for k in range(2, 10):
            r = rng.random()
            x[s, k] = 0.0 if r < 0.3 else (1.0 if r < 0.65 else -1.0) * 2.0 ** (tiny_e - int(rng.integers(0, 40)))
        if fill == "pairs":
            p = rng.standard_normal((L - 10) // 2) * 2.0 ** (e - 5)
            x[s, 10:] = np.concatenate([p, -p])
    x = x.reshape(-1)
    x[~np.isfinite(x)] = 0.0
    d = torch.from_numpy(x).cuda()
    b64, b32, fl, _ = oracle.sum_segments(x, seg_len=L)
    v, _, f = xs.sum_segments(d, L, flags=True)
    assert (v.cpu().numpy().view(np.uint64) == b64).all()
    assert (f.cpu().numpy().astype(np.uint32) == fl).all()
    v2, _, _ = xs.sum_segments(d, L)
    assert (v2.cpu().numpy().view(np.uint64) == b64).all()


def test_csr_segments_values_only_bands(xs):
    """K6's values-only CSR epilogue (one row per lane, the whole warp as one slot of band_round.cuh)
    and its fallbacks (exponents reaching row 31, NaN / Inf rescans, canonical images): ragged CSR
    segments (empty, single elements, partial tiles, > 8K) with a different exponent band in each;
    value and flags of every segment vs the oracle, and the same values with images requested."""
    import torch
    rng = np.random.default_rng(4242)
    lens = np.concatenate([[0, 1, 2, 255, 256, 257, 9000], rng.integers(0, 3000, 150)])
    rng.shuffle(lens)
    full = _band_segments(rng, lens.size, 9000).reshape(lens.size, 9000)   # every kind, cut to length
    x = np.concatenate([full[s, :int(L)] for s, L in enumerate(lens)])
    off = np.zeros(lens.size + 1, dtype=np.int64)
    off[1:] = np.cumsum(lens)
    d = to_dev(x, 0)
    o = torch.from_numpy(off).cuda()
    vals, _, flags = xs.sum_segments_csr(d, o, flags=True)
    b64, _, fl, _ = oracle.sum_segments(x, offsets=off)
    assert (vals.cpu().numpy().view(np.uint64) == b64).all()
    assert (flags.cpu().numpy().astype(np.uint32) == fl).all()
    vals2, _, _ = xs.sum_segments_csr(d, o, canon=True)
    assert (vals2.cpu().numpy().view(np.uint64) == b64).all()
