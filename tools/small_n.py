"""Small-n latency probe: back-to-back fused sums (GPU-bound average) and a CUDA-graph replay,
against an empty-ish torch kernel (development tool)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_05436_b200 as xsum  # noqa: E402
import synth  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "f64"
if kind == "f64":
    x_all = synth.device_generate("c2")
else:
    x_all = synth.device_bits({"f32": "c2f32", "f16": "c2f16", "bf16": "c2bf16"}[kind])
acc = xsum.Accumulator()
for k in (10, 14, 16, 18, 20, 22, 24, 26, 28):
    x = x_all[: 1 << k].clone()
    for _ in range(5):
        acc.sum(x)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    R = 200
    t0 = time.perf_counter()
    a.record()
    for _ in range(R):
        acc.sum(x)
    b.record()
    torch.cuda.synchronize()
    cpu_us = (time.perf_counter() - t0) / R * 1e6
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        acc.sum(x)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(20):
                acc.sum(x)
    torch.cuda.synchronize()
    c, d = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c.record()
    for _ in range(10):
        g.replay()
    d.record()
    torch.cuda.synchronize()
    print(f"n=2^{k:2d}: back-to-back {a.elapsed_time(b) / R * 1e3:7.2f} us/launch (host {cpu_us:6.2f} us/call), "
          f"graph {c.elapsed_time(d) / 200 * 1e3:7.2f} us/launch")
y = torch.zeros(16, device="cuda")
a.record()
for _ in range(200):
    y.add_(1)
b.record()
torch.cuda.synchronize()
print(f"torch add_ on 16 elements: {a.elapsed_time(b) / 200 * 1e3:.2f} us/launch")
