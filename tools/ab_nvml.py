"""A/B: does NVML clock polling during the timed region perturb the kernel time?"""
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1605_05436_b200 as xsum  # noqa: E402
import synth  # noqa: E402
from bench import ClockSampler  # noqa: E402

x = synth.device_generate("c2")
acc = xsum.Accumulator()
for _ in range(10):
    acc.sum(x)
torch.cuda.synchronize()


def run(K, sampler_period=None):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    cs = ClockSampler(0, sampler_period) if sampler_period else None
    if cs:
        cs.__enter__()
    for a, b in ev:
        a.record()
        acc.sum(x)
        b.record()
    torch.cuda.synchronize()
    if cs:
        cs.__exit__()
    per = [a.elapsed_time(b) for a, b in ev]
    tot = ev[0][0].elapsed_time(ev[-1][1])
    return statistics.median(per) * 1e3, statistics.mean(per) * 1e3, tot / K * 1e3


for trial in range(3):
    for K in (50, 200, 1000):
        for period in (None, 0.002, 0.05):
            med, mean, tot = run(K, period)
            print(f"K={K:5d} sampler={period}  median {med:7.1f} us  mean {mean:7.1f} us  total/K {tot:7.1f} us",
                  flush=True)
