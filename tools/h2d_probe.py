"""Pinned host -> device copy bandwidth (the ceiling of bench.py's e2e number)."""
import time

import torch

n = 1 << 28
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for chunk in (8 << 20, 64 << 20, 128 << 20, 2 << 30):
    per = chunk // 8
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        for off in range(0, n, per):
            d[off:off + per].copy_(h[off:off + per], non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(f"H2D chunks of {chunk >> 20:5d} MiB: {8 * n / dt / 1e9:6.1f} GB/s")
