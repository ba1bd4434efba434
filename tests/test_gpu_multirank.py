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
