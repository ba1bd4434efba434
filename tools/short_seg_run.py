"""Throughput of many short equal segments (development tool): 2^28 doubles as segments of
length L (xsum_sum_segments, one warp per segment) for small L."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1605_05436_b200 as xsum  # noqa: E402
import synth  # noqa: E402


def t_ms(f, reps=10):
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        f()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


for name in ("c2", "c1x"):
    # c2: exponents over [-1000, 1000]; c1x: c1's narrow exponents [-10, 10] (2^20 repeated)
    x = synth.device_generate("c2") if name == "c2" else synth.device_generate("c1").repeat(1 << 8)
    for L in (4, 16, 64, 256, 1024, 4096):
        ms = t_ms(lambda: xsum.sum_segments(x, L))
        ms_dim = t_ms(lambda: xsum.exact_sum_dim(x.view(-1, L), 1))
        print(f"{name:4s} L={L:5d}: {x.numel() // L:9d} segments  {ms * 1e3:9.1f} us  "
              f"{x.numel() / ms / 1e6:7.1f} G doubles/s  (exact_sum_dim over the last dim: {ms_dim * 1e3:9.1f} us)",
              flush=True)
