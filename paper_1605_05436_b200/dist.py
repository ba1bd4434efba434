"""Multi-GPU exact sums: one process per GPU, NCCL over NVLink / NVSwitch.

The paper's single-round MapReduce (§6.1; Spark version
PAPER.md:1172-1189): every reducer (here: a GPU) sums its share exactly into one
superaccumulator, the fixed-size superaccumulators are shuffled (here: one NCCL
all-gather of the 384-byte state images), and the post-process
merges them and rounds (here: xsum_merge + xsum_finalize_round on every rank, so
all ranks hold the identical double). Exact addition is associative, so any
partition of the input is valid.
"""
from __future__ import annotations

from . import STATE_BYTES, Accumulator, peer_buffer_bytes


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced shard [start, stop) of n items for `rank` of `world`
    (the first n % world ranks get one extra item)."""
    if world <= 0 or not (0 <= rank < world) or n < 0:
        raise ValueError("bad shard arguments")
    q, r = divmod(n, world)
    start = rank * q + min(rank, r)
    return start, start + q + (1 if rank < r else 0)


def gather_states(state, group=None):
    """All-gather the fixed-size state image of every rank -> uint8 tensor [world*384].

    Pure torch.distributed plumbing (works with NCCL on GPUs and gloo on CPU)."""
    import torch
    import torch.distributed as dist

    if state.dtype != torch.uint8 or state.numel() != STATE_BYTES:
        raise ValueError("state must be a uint8 tensor of 384 bytes")
    world = dist.get_world_size(group)
    if dist.get_backend(group) == "gloo":
        # host-staged exchange (CPU process groups; tests run several ranks on one GPU this way)
        host = state.detach().to("cpu").contiguous()
        parts = [torch.empty_like(host) for _ in range(world)]
        dist.all_gather(parts, host, group=group)
        return torch.cat(parts).to(state.device)
    out = torch.empty(world * STATE_BYTES, dtype=torch.uint8, device=state.device)
    dist.all_gather_into_tensor(out, state.contiguous(), group=group)
    return out


def allreduce_exact(acc: Accumulator, group=None) -> Accumulator:
    """Replace acc's state by the exact sum of all ranks' states (identical on every rank)."""
    states = gather_states(acc.state, group)
    acc.reset()
    acc.merge(states)
    return acc


def exact_sum_distributed(x, acc: Accumulator, total: Accumulator, group=None, out=None):
    """The whole multi-GPU step on this rank's shard x: local fused sum (one launch), NCCL
    all-gather of the 384-byte states, fused merge + round (one launch). Returns the device
    result record (in `out` if given); every rank gets the identical bits."""
    acc.sum(x)                                   # state := sum(x) (its local rounding is unused)
    states = gather_states(acc.state, group)
    res, _ = total.merge_round(states, out=out)
    return res


class PeerExchange:
    """Exchange buffers of the fused multi-GPU step (xsum_sum_allreduce): one per rank, mapped
    into every rank's address space through torch symmetric memory (CUDA IPC over NVLink), zeroed
    once; `epoch` counts the calls made on them (the kernel's arrival counters are monotone).

    The step is ONE launch per rank: the shard's fused sum, then the last block publishes the
    state to every peer (P2P stores), signals, waits for all and merges -
    no NCCL call on the data path."""

    def __init__(self, device, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        self.group = group if group is not None else dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        nbytes = peer_buffer_bytes(self.world)
        # a rank that cannot allocate its buffer must not leave the others blocked in the
        # (collective) rendezvous: agree first, then every rank raises or every rank proceeds
        ok = torch.ones(1, dtype=torch.int32, device=device)
        err = None
        try:
            self.buf = symm_mem.empty(nbytes, dtype=torch.uint8, device=device)
            self.buf.zero_()
        except Exception as e:  # noqa: BLE001
            err = e
            ok.zero_()
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=self.group)
        if not int(ok.item()):
            raise RuntimeError(f"symmetric peer buffers unavailable on some rank (this rank: {err!r})")
        torch.cuda.synchronize(device)
        self.handle = symm_mem.rendezvous(self.buf, self.group.group_name)
        self.bufs_dev = int(self.handle.buffer_ptrs_dev)
        self.epoch = 0
        dist.barrier(group=self.group)

    def sum(self, x, acc: Accumulator, canon: bool = False, out=None):
        """State of `acc` := exact sum over all ranks' shards x (one launch); returns the device
        (result, canon), bit-identical on every rank (the result record in `out` if given)."""
        self.epoch += 1
        return acc.sum_allreduce(x, self.bufs_dev, self.rank, self.world, self.epoch, canon=canon, out=out)
