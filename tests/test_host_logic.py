"""CPU-side checks of the boundary and host logic (no GPU needed):
the C-ABI library loads and exports every symbol include/xsum.h declares, the
state/result layouts match the header, the headroom bound behind the kernel's
flush schedule holds, shard partitioning, and the multi-rank state exchange
(world_size 2 over gloo)."""
from __future__ import annotations

import ctypes
import os
import re
import subprocess
import sys

import numpy as np
import pytest

import paper_1605_05436_b200 as xsum
from paper_1605_05436_b200 import dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "xsum.h")


def header_functions() -> list[str]:
    text = open(HEADER).read()
    return sorted(set(re.findall(r"XSUM_API\s+[\w\s\*]+?\b(xsum_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def built():
    xsum.build()
    return xsum.lib()


def test_header_declares_the_north_star_calls():
    fns = header_functions()
    for f in ("xsum_create", "xsum_accumulate", "xsum_merge", "xsum_finalize_round", "xsum_destroy"):
        assert f in fns
    assert set(fns) == set(xsum.EXPORTS)


def test_library_exports_every_header_symbol(built):
    out = subprocess.run(["nm", "-D", "--defined-only", xsum.SO_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\sT\s(xsum_\w+)", out))
    assert set(header_functions()) <= exported
    # nothing but the C-ABI is exported (kernels and helpers stay hidden)
    assert {s for s in exported if s.startswith("xsum_")} == set(header_functions())


def test_pdl_kernels_load_no_input_before_griddepcontrol_wait(built):
    """Every kernel that waits on its programmatic predecessor (griddepcontrol.wait = SASS ACQBULK)
    issues no global load ahead of the first wait in its SASS and uses no non-coherent
    (LDG.CONSTANT) loads: ptxas schedules ld.global.nc above the wait (ADVICE r01 PDL finding;
    the GPU counterpart is test_pdl_consumer_waits_for_an_early_triggering_producer)."""
    sass = subprocess.run(["cuobjdump", "-sass", xsum.SO_PATH], capture_output=True, text=True).stdout
    if not sass:
        pytest.skip("cuobjdump unavailable")
    funcs = re.split(r"\n\s*Function : ", sass)[1:]
    waiting = 0
    for f in funcs:
        name, body = f.split("\n", 1)
        if "ACQBULK" not in body:
            continue
        waiting += 1
        before = body.split("ACQBULK", 1)[0]
        assert not re.search(r"\bLDG", before), f"{name}: global load before griddepcontrol.wait"
        assert not re.search(r"LDG[^;]*CONSTANT", body), f"{name}: non-coherent input load"
    assert waiting >= 4            # K2, K2f, K2h (binary16, bfloat16)


def test_library_sizes_match_header(built):
    L = built
    assert L.xsum_state_bytes() == xsum.STATE_BYTES == 384
    assert L.xsum_result_bytes() == xsum.RESULT_BYTES == 48
    # arrival counter (0), flags word (4), grid accumulator of 42 u64 digits at byte 256
    assert L.xsum_scratch_bytes(0) >= 256 + 8 * 42
    assert L.xsum_status_str(0) == b"ok"
    assert L.xsum_status_str(2).startswith(b"capacity")


def test_host_side_argument_errors_without_gpu(built):
    """Argument checks run on the host before anything touches the device."""
    L = built
    assert L.xsum_accumulate(None, None, 5, None) == xsum.EINVAL
    assert L.xsum_merge(None, None, 1, None) == xsum.EINVAL
    assert L.xsum_finalize_round(None, None, None, None) == xsum.EINVAL
    assert L.xsum_destroy(None) == xsum.EINVAL
    assert L.xsum_count(None) == 0
    assert L.xsum_sum_segments(None, 0, 10, None, None, None, None) == xsum.OK      # nothing to do
    assert L.xsum_sum_segments(None, 4, 10, None, None, None, None) == xsum.EINVAL  # null output
    h = ctypes.c_void_p()
    rc = L.xsum_create(ctypes.byref(h), 0, None, None, 0, None)
    assert rc in (xsum.EINVAL, xsum.ECUDA) and not h.value


def test_header_struct_layout_by_compiling_it(tmp_path):
    """offsets of the state image / result record, checked by the C compiler itself."""
    src = tmp_path / "layout.c"
    src.write_text(r'''
#include <stddef.h>
#include <stdio.h>
#include "xsum.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu\n", sizeof(xsum_state_image), offsetof(xsum_state_image, digit),
         offsetof(xsum_state_image, count), sizeof(xsum_result), offsetof(xsum_result, sig53),
         offsetof(xsum_result, count));
  return 0;
}''')
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    vals = [int(v) for v in subprocess.check_output([str(exe)]).split()]
    assert vals == [384, 24, 16, 48, 32, 24]


def test_result_record_parsing():
    rec = np.zeros(48, dtype=np.uint8)
    rec[0:8] = np.array([1.5], dtype=np.float64).view(np.uint8)
    rec[8:12] = np.array([-1], dtype=np.int32).view(np.uint8)
    rec[12:16] = np.array([16], dtype=np.uint32).view(np.uint8)
    rec[16:20] = np.array([-(2 ** 31)], dtype=np.int32).view(np.uint8)
    rec[24:32] = np.array([7], dtype=np.uint64).view(np.uint8)
    r = xsum.Result.from_bytes(rec.tobytes())
    assert r.value == 1.5 and r.direction == -1 and r.flags == 16 and r.msb_exp is None and r.count == 7


def test_digit_index_division_and_chunk_split_cover_binary64():
    """Arithmetic facts the kernel relies on, over all exponents:
    k = max(e,1)-1 in [0,2045] -> digit i = k//52 <= 39, so chunks land in digits <= 40 < 42,
    and the two chunks of M*2^o (o = k mod 52) are < 2^52 in magnitude."""
    for e in range(0, 2047):
        k = max(e, 1) - 1
        i, o = divmod(k, 52)
        assert i + 1 <= 40
        M = (1 << 53) - 1
        v = M << o
        c0, c1 = v & ((1 << 52) - 1), v >> 52
        assert c0 < 2 ** 52 and c1 < 2 ** 52
        c1n = (-M << o) >> 52                  # arithmetic floor for the negative case
        assert -(2 ** 52) <= c1n < 0
    # digits: 42 * 52 = 2184 bits >= 1074 + 1024 + 63 (n < 2^63 summands)
    assert 42 * 52 >= 1074 + 1024 + 63
    assert 34 * 64 >= 1074 + 1024 + 63 + 1


def test_flush_headroom_bound():
    """FLUSH_ELEMS: residue + (F + 17 stragglers) chunk adds + the balanced-carry offset fit
    int64; the NaN/Inf compensation window (<= F adds after a regularization) likewise."""
    src = open(os.path.join(ROOT, "paper_1605_05436_b200", "csrc", "xsum_device.cuh")).read()
    F = int(re.search(r"FLUSH_ELEMS = (\d+)", src).group(1))
    assert F % 16 == 0                                   # whole tiles (8 binary64 / 16 binary32 per lane)
    residue = 2 ** 51 + 2 ** 11
    worst = residue + (F + 17) * 2 ** 52
    assert worst + 2 ** 51 < 2 ** 63
    assert residue + F * 2 ** 52 + 2 ** 51 < 2 ** 63   # compensation window
    # balanced carry magnitude after a window, and the block/grid raw sums
    assert (worst + 2 ** 51) >> 52 <= 2 ** 11
    assert 512 * (2 ** 51 + 2 ** 11) < 2 ** 63          # block sum of 512 regularized lane columns
    assert 1024 * (2 ** 51 + 2 ** 9) + 2 ** 52 < 2 ** 62  # grid sum of <= XS_MAXB block partials + state


@pytest.mark.parametrize("n,world", [(0, 1), (10, 3), (2 ** 33, 8), (7, 8), (2 ** 28 + 2 ** 20, 4)])
def test_shard_range_partitions(n, world):
    spans = [dist.shard_range(n, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    for (a, b), (c, d) in zip(spans, spans[1:]):
        assert b == c
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1


def _gloo_worker(rank: int, world: int, port: int, q):
    import torch
    import torch.distributed as tdist

    import oracle
    import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 300_001
        a, b = dist.shard_range(n, rank, world)
        x = synth.gen.generate("c2", a, b - a)
        # the state image a rank would produce (built test-side from the oracle: value-equal
        # regularized digits with the header of include/xsum.h)
        r, limbs = oracle.exact_sum(x)
        img = encode_state(oracle.limbs_to_int(limbs), b - a)
        states = dist.gather_states(torch.from_numpy(img))
        q.put((rank, states.numpy().tobytes()))
    finally:
        tdist.destroy_process_group()


def encode_state(A: int, count: int, flags: int = 0) -> np.ndarray:
    """State image (include/xsum.h layout) holding the integer A in balanced radix-2^52 digits."""
    R = 1 << 52
    digits = []
    v = A
    for j in range(42):
        if j == 41:
            digits.append(v)
            break
        d = ((v + R // 2) % R) - R // 2
        digits.append(d)
        v = (v - d) // R
    img = np.zeros(384, dtype=np.uint8)
    img[0:4] = np.array([xsum.MAGIC], dtype=np.uint32).view(np.uint8)
    img[4:6] = np.array([1], dtype=np.uint16).view(np.uint8)
    img[6] = 52
    img[7] = 42
    img[8:12] = np.array([flags], dtype=np.uint32).view(np.uint8)
    img[16:24] = np.array([count], dtype=np.uint64).view(np.uint8)
    img[24:24 + 8 * 42] = np.array(digits, dtype=np.int64).view(np.uint8)
    return img


def decode_state(img: np.ndarray) -> tuple[int, int]:
    d = np.frombuffer(img[24:24 + 8 * 42].tobytes(), dtype=np.int64)
    return sum(int(v) << (52 * j) for j, v in enumerate(d)), int(np.frombuffer(img[16:24].tobytes(), np.uint64)[0])


def test_state_codec_roundtrip():
    for A in (0, 1, -1, (1 << 2000) - 12345, -(1 << 2100) + 7):
        assert decode_state(encode_state(A, 5)) == (A, 5)


def test_checkpoint_image_validation(built):
    """xsum_check_state_image (the gate of xsum_load_state): accepts every well-formed image,
    rejects each single header/range violation (include/xsum.h layout)."""
    R = 1 << 52
    for A, cnt, fl in ((0, 0, 0), (1, 1, 0), (-(1 << 2100) + 7, 2 ** 63 - 1, 0), ((1 << 1500) - 3, 9, 1 | 2 | 4)):
        assert xsum.check_state_image(encode_state(A, cnt, fl).tobytes())

    def bad(mut):
        img = encode_state(12345 << 700, 77)
        mut(img)
        return not xsum.check_state_image(img.tobytes())

    def setd(j, v):
        def f(img):
            img[24 + 8 * j:32 + 8 * j] = np.array([v], dtype=np.int64).view(np.uint8)
        return f

    assert bad(lambda i: i.__setitem__(0, 0))                               # magic
    assert bad(lambda i: i.__setitem__(4, 2))                               # version
    assert bad(lambda i: i.__setitem__(6, 51))                              # radix
    assert bad(lambda i: i.__setitem__(7, 44))                              # digit count
    assert bad(lambda i: i.__setitem__(12, 1))                              # reserved word
    assert bad(lambda i: i.__setitem__(383, 1))                             # padding
    assert bad(lambda i: i.__setitem__(9, 1))                               # unknown flag bit 256
    assert bad(lambda i: i.__setitem__(23, 0x80))                           # count >= 2^63
    assert bad(setd(3, R))                                                  # |digit| > R-1
    assert bad(setd(40, -R))
    assert bad(setd(41, (1 << 29) + 1))                                     # top digit bound
    assert not bad(setd(3, R - 1)) and not bad(setd(3, -(R - 1))) and not bad(setd(41, -(1 << 29)))
    assert not xsum.check_state_image(b"\0" * 383)


def test_two_rank_gloo_state_exchange():
    """world_size 2: every rank receives every rank's state image; merging the gathered
    images (decoded here) gives the exact sum of the whole input."""
    import multiprocessing as mp

    import oracle
    import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 2000)
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got[0] == got[1]
    blob = np.frombuffer(got[0], dtype=np.uint8)
    total, cnt = 0, 0
    for r in range(2):
        A, c = decode_state(blob[r * 384:(r + 1) * 384])
        total += A
        cnt += c
    _, limbs = oracle.exact_sum(synth.gen.generate("c2", 0, 300_001))
    assert total == oracle.limbs_to_int(limbs) and cnt == 300_001


def test_product_package_never_imports_oracle():
    """The CUDA path and the oracle share no code: no product module imports oracle/."""
    pkg = os.path.join(ROOT, "paper_1605_05436_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".c", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", text, re.M), f
                assert "xsum_oracle" not in text and "pytwin" not in text, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c")):
            text = open(os.path.join(ROOT, "oracle", f)).read()
            assert not re.search(r"^\s*(import|from)\s+paper_1605_05436_b200", text, re.M), f
            assert not re.search(r'#include\s+"xsum', text), f


def test_decode_magic_constants():
    """Constants of decompose() in xsum_device.cuh: mulhi(k, K52) = k // 52 for every
    k the kernels can see (k <= 2046 for binary64, <= 1194 for the other formats; 0..2047 checked)."""
    src = open(os.path.join(ROOT, "paper_1605_05436_b200", "csrc", "xsum_device.cuh")).read()
    k52 = eval(re.search(r"constexpr uint32_t K52 = (.*?);", src).group(1).replace("u", ""))
    for k in range(2048):
        assert (k * k52) >> 32 == k // 52
    # dec3 tracks NaN/Inf by max(k): k = max(e,1)-1 reaches 2046 only for e = 2047
    assert max(max(e, 1) - 1 for e in range(2047)) == 2045 and max(2047, 1) - 1 == 2046
    # hi - k*2^20 keeps the sign bit and sets the hidden bit exactly when e != 0
    for e in (0, 1, 2, 1023, 2046, 2047):
        for s in (0, 1):
            m_hi = 0xABCDE
            hi = (s << 31) | (e << 20) | m_hi
            k = max(e, 1) - 1
            mhs = (hi - k * (1 << 20)) & 0xFFFFFFFF
            assert mhs == (s << 31) | ((1 if e else 0) << 20) | m_hi


def test_sparse_image_decoder_on_a_hand_built_image():
    """The sparse wire format of include/xsum.h, built byte by byte: header then records
    (digit << 6) | index; digit -3 at index 20 and 2^51 at index 21 (value -3 R^20 + 2^51 R^21)."""
    import struct

    import paper_1605_05436_b200 as xs
    hdr = struct.pack("<IHBBIIQ", 0x41505358, 1, 52, 2, 4, 0, 12345)
    recs = struct.pack("<qq", (-3 << 6) | 20, ((1 << 51) << 6) | 21)
    d = xs.decode_sparse(hdr + recs)
    assert d == {"flags": 4, "count": 12345, "digits": {20: -3, 21: 1 << 51}}
    assert xs.SPARSE_MAX_BYTES == 24 + 8 * 42
    import pytest
    with pytest.raises(ValueError):
        xs.decode_sparse(struct.pack("<IHBBIIQ", 0x41505359, 1, 52, 0, 0, 0, 0))   # bad magic
    with pytest.raises(ValueError):
        xs.decode_sparse(hdr + recs[:8])                                          # truncated


def _result_bytes(bits: int, flags: int):
    import torch
    a = np.zeros(xsum.RESULT_BYTES, dtype=np.uint8)
    a[0:8] = np.array([bits], dtype=np.uint64).view(np.uint8)
    a[12:16] = np.array([flags], dtype=np.uint32).view(np.uint8)
    return torch.from_numpy(a)


def _fused_check_worker(rank: int, world: int, port: int, mode: str, q):
    """bench.fused_check with stand-ins for the fused step (pe.sum) and the NCCL path
    (dist.exact_sum_distributed): CPU tensors, gloo group."""
    import types

    import torch
    import torch.distributed as tdist
    sys.path.insert(0, ROOT)
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        good = 0x3FF0000000000001
        fused_bits, fused_flags = good, 0
        if mode == "timeout":
            fused_flags = xsum.F_PEER_TIMEOUT
        elif mode == "one_rank_wrong" and rank == 1:
            fused_bits = good ^ 1
        pe = types.SimpleNamespace(sum=lambda x, acc: (_result_bytes(fused_bits, fused_flags), None))
        fake_dist = types.SimpleNamespace(exact_sum_distributed=lambda x, acc, tot: _result_bytes(good, 0))
        fake_xsum = types.SimpleNamespace(Result=xsum.Result, F_PEER_TIMEOUT=xsum.F_PEER_TIMEOUT,
                                          Accumulator=lambda device: None)
        why = bench.fused_check(fake_xsum, fake_dist, pe, torch.zeros(10, dtype=torch.float64), None, None)
        q.put((rank, why))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("mode", ["ok", "timeout", "one_rank_wrong"])
def test_bench_fused_check_two_ranks(mode):
    """bench.py times the fused multi-GPU step only if every rank's fused result on a probe
    equals the NCCL all-gather path's with no peer timeout; one rank's disagreement makes every
    rank fall back (the decision is all-reduced)."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31500 + (os.getpid() % 2000) + ["ok", "timeout", "one_rank_wrong"].index(mode) * 7
    procs = [ctx.Process(target=_fused_check_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    if mode == "ok":
        assert got == {0: None, 1: None}
    else:
        assert got[0] is not None and got[1] is not None
        if mode == "one_rank_wrong":
            assert got[0] == "another rank disagreed" and got[1].startswith("rank result")


def _rows(bits_flags):
    return np.stack([_result_bytes(b, f).numpy() for b, f in bits_flags])


def _steps_verdict_worker(rank: int, world: int, port: int, mode: str, q):
    """bench.steps_verdict over gloo on CPU: every rank checks its K timed results; the decision
    is all-reduced."""
    import torch
    import torch.distributed as tdist
    sys.path.insert(0, ROOT)
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        good = 0x3FF0000000000001
        steps = [(good, 0)] * 4
        if mode == "timeout_mid" and rank == 1:
            steps = [(good, 0), (good ^ 8, xsum.F_PEER_TIMEOUT), (good, 0), (good, 0)]   # not the last step
        elif mode == "drift" and rank == 0:
            steps = [(good, 0), (good, 0), (good ^ 1, 0), (good, 0)]
        elif mode == "disagree" and rank == 1:
            steps = [(good ^ 2, 0)] * 4
        q.put((rank, bench.steps_verdict(xsum, _rows(steps), world, torch.device("cpu"))))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("mode", ["ok", "timeout_mid", "drift", "disagree"])
def test_bench_steps_verdict_two_ranks(mode):
    """bench.py checks EVERY timed step's result record on every rank: a
    peer timeout in a middle step, results that change between steps, or ranks that disagree
    invalidate the region on all ranks (the fused region is then re-timed on the NCCL path)."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    modes = ["ok", "timeout_mid", "drift", "disagree"]
    port = 33600 + (os.getpid() % 2000) + modes.index(mode) * 7
    procs = [ctx.Process(target=_steps_verdict_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    if mode == "ok":
        assert got == {0: None, 1: None}
    elif mode == "timeout_mid":
        assert got[1].startswith("peer timeout in timed step(s) [1]")
        assert got[0] == "peer timeout in a timed step on another rank"
    elif mode == "drift":
        assert got[0] == got[1] == "results differ between timed steps"
    else:
        assert got[0] == got[1] == "ranks disagree on the result"


def test_xsum_library_override_needs_dev_flag():
    """A stray XSUM_LIBRARY must not swap the library under test."""
    code = ("import paper_1605_05436_b200 as x, os; "
            "print(os.path.basename(os.path.dirname(x.SO_PATH)) + '/' + os.path.basename(x.SO_PATH))")
    env = dict(os.environ, XSUM_LIBRARY="/nonexistent/libother.so")
    env.pop("XSUM_DEV", None)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=ROOT)
    assert out.stdout.strip() == "paper_1605_05436_b200/libxsum.so", out.stderr
    env["XSUM_DEV"] = "1"
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=ROOT)
    assert out.stdout.strip() == "nonexistent/libother.so", out.stderr
