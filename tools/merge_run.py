"""Latency of the post-process merges (development tool): xsum_merge_round of p dense state
images, xsum_merge_sparse of p sparse images, and the fused-exchange protocol with virtual ranks
(xsum_peer_selftest, one cooperative launch), CUDA-graph replayed / event-timed."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1605_05436_b200 as xsum  # noqa: E402
import synth  # noqa: E402


def timeit(f, reps=200):
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


x = synth.device_generate("c2")[: 1 << 22].clone()
for p in (2, 8, 64, 1024):
    cuts = [x.numel() * i // p for i in range(p + 1)]
    states = torch.cat([xsum.Accumulator().add(x[cuts[i]:cuts[i + 1]]).state for i in range(p)])
    tot = xsum.Accumulator()
    us = timeit(lambda: tot.merge_round(states))
    imgs, offs, o = [], [], 0
    for i in range(p):
        a = xsum.Accumulator()
        a.merge(states[i * 384:(i + 1) * 384].clone())
        img, nb = a.to_sparse()
        imgs.append(img.cpu().numpy())
        offs.append(o)
        o += nb
    blob = torch.from_numpy(np.concatenate(imgs)).cuda()
    offt = torch.tensor(offs, dtype=torch.int64, device="cuda")
    sp = xsum.Accumulator()
    us_sp = timeit(lambda: sp.reset().merge_sparse(blob, offt))
    print(f"p={p:5d}: merge_round of dense images {us:7.2f} us; reset + merge_sparse {us_sp:7.2f} us "
          f"(sparse bytes {o}, dense {384 * p})", flush=True)
for world in (2, 8):
    st = torch.cat([xsum.Accumulator().add(x[: 1 << 20]).state for _ in range(world)])
    bufs = None
    ep = [0]

    def one():
        global bufs
        ep[0] += 1
        _, _, bufs = xsum.peer_selftest(st, world, ep[0], bufs)
    print(f"peer exchange protocol, {world} virtual ranks in one launch (incl. host result copy): "
          f"{timeit(one, 50):.1f} us", flush=True)
