"""How the timing method moves the c2 number (development tool): 200 back-to-back fused sums
bracketed by one event pair, with and without the NVML clock sampler running, and per-step
events (median and mean)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1605_05436_b200 as xsum  # noqa: E402
import synth  # noqa: E402

x = synth.device_generate("c2")
acc = xsum.Accumulator()
K = 200
for _ in range(10):
    acc.sum(x)
torch.cuda.synchronize()


def span(sampler: bool) -> float:
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if sampler:
        with bench.ClockSampler(0):
            a.record()
            for _ in range(K):
                acc.sum(x)
            b.record()
            torch.cuda.synchronize()
    else:
        a.record()
        for _ in range(K):
            acc.sum(x)
        b.record()
        torch.cuda.synchronize()
    return a.elapsed_time(b) / K * 1e3


def per_step():
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    torch.cuda.synchronize()
    for a, b in ev:
        a.record()
        acc.sum(x)
        b.record()
    torch.cuda.synchronize()
    t = [a.elapsed_time(b) * 1e3 for a, b in ev]
    return statistics.median(t), statistics.mean(t), max(t), min(t)


for rep in range(3):
    s0 = span(False)
    s1 = span(True)
    med, mean, mx, mn = per_step()
    g = lambda us: x.numel() / us / 1e3  # noqa: E731
    print(f"rep {rep}: span/K no sampler {s0:.1f} us ({g(s0):.0f} G/s); with sampler {s1:.1f} us ({g(s1):.0f}); "
          f"per-step median {med:.1f} mean {mean:.1f} min {mn:.1f} max {mx:.1f} us ({g(med):.0f} / {g(mean):.0f})",
          flush=True)
