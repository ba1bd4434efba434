"""The multi-GPU step (dist.exact_sum_distributed) end to end with two ranks on ONE GPU: each
rank sums its shard with the fused kernel, the 384-byte states are exchanged over a gloo
(host-staged) process group instead of NCCL, and every rank runs xsum_merge_round. No kernel
waits on another rank, so sharing one GPU is safe (B200_PROFILING.md's rule concerns kernels
that spin on each other). Every rank must hold the identical, oracle-exact result."""
from __future__ import annotations

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rank(rank: int, world: int, port: int, n: int, q):
    import torch
    import torch.distributed as tdist

    import paper_1605_05436_b200 as xsum
    import synth
    from paper_1605_05436_b200 import dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        a, b = dist.shard_range(n, rank, world)
        x = synth.device_generate("c4", a, b - a, device="cuda:0")
        acc, tot = xsum.Accumulator("cuda:0"), xsum.Accumulator("cuda:0")
        res = dist.exact_sum_distributed(x, acc, tot)
        r = xsum.Result.from_bytes(res.cpu().numpy().tobytes())
        _, canon = tot.exact()
        q.put((rank, r.bits, r.flags, r.count, canon.tobytes()))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_step_two_ranks_one_gpu(world):
    import multiprocessing as mp

    import oracle
    import synth
    n = 4_000_037
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31000 + (os.getpid() % 1000) + 10 * world
    procs = [ctx.Process(target=_rank, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref, limbs = oracle.exact_sum(synth.gen.generate("c4", 0, n))
    for rank, bits, flags, count, canon in got:
        assert bits == ref.bits and flags == ref.flags and count == n, rank
        assert (np.frombuffer(canon, dtype=np.uint64) == limbs).all(), rank


# ------------------------------------------------------------------------------------------
# fused multi-GPU step: the exchange protocol with virtual ranks in ONE cooperative launch
# (one block per rank, all co-resident), the B200_PROFILING.md way of testing kernels that
# wait on one another with fewer GPUs than ranks.
# ------------------------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_peer_exchange_protocol_virtual_ranks(world):
    import numpy as np
    import torch

    import oracle
    import paper_1605_05436_b200 as xsum
    import synth
    xsum.build()
    n = 3_000_017
    x = synth.gen.generate("c4", 5, n)
    cuts = [n * r // world for r in range(world + 1)]
    states = []
    for r in range(world):
        acc = xsum.Accumulator().add(torch.from_numpy(x[cuts[r]:cuts[r + 1]]).cuda())
        states.append(acc.state.clone())
    st = torch.cat(states)
    ref, limbs = oracle.exact_sum(x)
    bufs = None
    for epoch in (1, 2, 3):                           # repeated calls: epoch parity slots, monotone counters
        res, out, bufs = xsum.peer_selftest(st, world, epoch, bufs)
        imgs = out.cpu().numpy().reshape(world, -1)
        for r in range(world):
            assert res[r].bits == ref.bits and res[r].flags == ref.flags and res[r].count == n, (world, epoch, r)
            assert (imgs[r] == imgs[0]).all()         # bit-identical digits on every rank
        m = xsum.Accumulator().merge(out[:384].clone())
        _, canon = m.exact()
        assert (canon == limbs).all()


@pytest.mark.gpu
def test_fused_allreduce_single_rank_world():
    """xsum_sum_allreduce with world = 1 (its own buffer as the only peer): the fused kernel's
    exchange path end to end on the real accumulate launch."""
    import torch

    import oracle
    import paper_1605_05436_b200 as xsum
    import synth
    xsum.build()
    x = synth.gen.generate("c2", 8, 2_000_003)
    buf = torch.zeros(xsum.peer_buffer_bytes(1), dtype=torch.uint8, device="cuda")
    ptrs = torch.tensor([buf.data_ptr()], dtype=torch.int64, device="cuda")
    acc = xsum.Accumulator()
    ref, limbs = oracle.exact_sum(x)
    d = torch.from_numpy(x).cuda()
    for epoch in (1, 2, 3, 4):
        res, canon = acc.sum_allreduce(d, ptrs.data_ptr(), 0, 1, epoch, canon=True)
        r = xsum.Result.from_bytes(res.cpu().numpy().tobytes())
        assert r.bits == ref.bits and r.flags == ref.flags and r.count == x.size
        assert (canon.cpu().numpy().view("u8") == limbs).all()
    # a missing peer (world 2, nobody else calls) times out instead of hanging
    b2 = [torch.zeros(xsum.peer_buffer_bytes(2), dtype=torch.uint8, device="cuda") for _ in range(2)]
    ptrs2 = torch.tensor([b.data_ptr() for b in b2], dtype=torch.int64, device="cuda")
    res, _ = acc.sum_allreduce(d, ptrs2.data_ptr(), 0, 2, 1)
    r = xsum.Result.from_bytes(res.cpu().numpy().tobytes())
    assert r.flags & xsum.F_PEER_TIMEOUT


def _symm_rank(port: int, q):
    import torch
    import torch.distributed as tdist

    import oracle
    import paper_1605_05436_b200 as xsum
    import synth
    from paper_1605_05436_b200 import dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    tdist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        x = synth.gen.generate("c2", 11, 1_000_003)
        ref, limbs = oracle.exact_sum(x)
        d = torch.from_numpy(x).cuda()
        pe = dist.PeerExchange(torch.device("cuda", 0))      # torch symmetric memory + rendezvous
        acc = xsum.Accumulator()
        ok = []
        for _ in range(3):                                     # consecutive epochs on the same buffers
            res, canon = pe.sum(d, acc, canon=True)
            r = xsum.Result.from_bytes(res.cpu().numpy().tobytes())
            ok.append(r.bits == ref.bits and r.flags == ref.flags and
                      bool((canon.cpu().numpy().view("u8") == limbs).all()))
        # the NCCL fallback path on the same group
        tot = xsum.Accumulator()
        r2 = xsum.Result.from_bytes(dist.exact_sum_distributed(d, xsum.Accumulator(), tot).cpu().numpy().tobytes())
        ok.append(r2.bits == ref.bits and r2.flags == ref.flags)
        q.put(("ok", ok))
    except Exception as e:  # noqa: BLE001
        q.put(("error", repr(e)))
    finally:
        tdist.destroy_process_group()


@pytest.mark.gpu
def test_peer_exchange_symmetric_memory_nccl_world1():
    """The bench's N > 1 setup on the real stack: an NCCL process group, dist.PeerExchange
    (torch symmetric memory allocation + rendezvous, device pointer table) and the fused
    one-launch step through it, three epochs, plus the NCCL all-gather path; world size 1 (one
    GPU), so no kernel waits on another process."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_symm_rank, args=(29700 + os.getpid() % 1000, q))
    p.start()
    kind, val = q.get(timeout=300)
    p.join(timeout=60)
    assert kind == "ok", val
    assert all(val), val


# ------------------------------------------------------------------------------------------
# full-size sharded c4: exactly the arithmetic of the N = 2/4/8 bench run
# (contiguous shards of dist.shard_range, one fused xsum_sum per shard, the 384-byte states
# merged by xsum_merge_round) at 2^33 doubles, on one GPU; the fused-exchange
# protocol runs on the same p states with p virtual ranks.
# ------------------------------------------------------------------------------------------
@pytest.fixture(scope="module")
def c4_oracle_eighths():
    """The oracle's exact sums of the 8 contiguous eighths of c4 (streamed from the host
    generator); coarser shards are their exact merges (oracle limb addition)."""
    import oracle
    import synth
    from paper_1605_05436_b200 import dist
    n = synth.CONFIGS["c4"]["n"]
    chunk = 1 << 26
    buf = np.empty(chunk, dtype=np.float64)
    parts = []
    for r in range(8):
        a, b = dist.shard_range(n, r, 8)
        acc = oracle.Accumulator()
        for s in range(a, b, chunk):
            c = min(chunk, b - s)
            acc.add(synth.host_generate("c4", s, c, out=buf[:c]))
        parts.append(acc)
    return parts


@pytest.mark.slow
@pytest.mark.parametrize("p", [2, 4, 8])
def test_full_c4_sharded_merge(c4_oracle_eighths, p):
    import torch

    import oracle
    import paper_1605_05436_b200 as xsum
    import synth
    from paper_1605_05436_b200 import dist
    xsum.build()
    cfg = synth.CONFIGS["c4"]
    n = cfg["n"]
    free, _ = torch.cuda.mem_get_info()
    if free < n * 8 // p + (4 << 30):
        pytest.skip("not enough device memory for one shard")
    # the oracle of each of the p shards (merged eighths) and of the whole
    per = 8 // p
    shard_ref = []
    for r in range(p):
        o = oracle.Accumulator()
        for k in range(r * per, (r + 1) * per):
            o.merge(c4_oracle_eighths[k])
        shard_ref.append(o)
    whole = oracle.Accumulator()
    for o in shard_ref:
        whole.merge(o)
    ref, limbs = whole.result(), whole.limbs.copy()
    states = []
    buf = torch.empty(n // p + 1, dtype=torch.float64, device="cuda")
    for r in range(p):
        a, b = dist.shard_range(n, r, p)
        x = synth.device_generate("c4", a, b - a, device="cuda", out=buf[: b - a])
        acc = xsum.Accumulator()
        res, canon = acc.sum(x, canon=True)                 # the bench's per-rank fused launch
        rr = xsum.Result.from_bytes(res.cpu().numpy().tobytes())
        sr = shard_ref[r].result()
        assert rr.bits == sr.bits and rr.flags == sr.flags and rr.count == b - a, (p, r)
        assert (canon.cpu().numpy().view(np.uint64) == shard_ref[r].limbs).all(), (p, r)
        states.append(acc.state.clone())
    del buf
    torch.cuda.empty_cache()
    st = torch.cat(states)
    tot = xsum.Accumulator()
    res, canon = tot.merge_round(st, canon=True)           # the NCCL path's post-process
    rr = xsum.Result.from_bytes(res.cpu().numpy().tobytes())
    assert rr.bits == ref.bits and rr.flags == ref.flags and rr.count == n and rr.sig53 == ref.sig53 \
        and rr.exp2 == ref.exp2
    assert (canon.cpu().numpy().view(np.uint64) == limbs).all()
    assert tot.count == n
    # the fused exchange protocol on the same p states (p virtual ranks, one cooperative launch)
    results, out, _ = xsum.peer_selftest(st, p, 1)
    imgs = out.cpu().numpy().reshape(p, -1)
    for r in range(p):
        assert results[r].bits == ref.bits and results[r].flags == ref.flags and results[r].count == n, (p, r)
        assert (imgs[r] == imgs[0]).all()
    m = xsum.Accumulator().merge(out[:384].clone())
    _, canon2 = m.exact()
    assert (canon2 == limbs).all()
