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

# ragged CSR segments, mostly short (sparse-matrix-like rows): K11c (the binding's choice for a mean
# length <= 256) vs the warp-per-segment path with the ticket order (xsum_sum_segments_ws)
import numpy as np  # noqa: E402

x = synth.device_generate("c5")
for maxlen in (8, 32, 128, 512):
    rng = np.random.default_rng(maxlen)
    nseg = int(x.numel() // (maxlen / 2 + 0.5))
    lens = rng.integers(0, maxlen + 1, size=nseg)
    offs = np.concatenate([[0], np.cumsum(lens)])
    keep = int(np.searchsorted(offs, x.numel(), side="right")) - 1
    offs_t = torch.from_numpy(offs[:keep + 1].astype(np.int64)).cuda()
    n = int(offs[keep])
    out = torch.empty(keep, dtype=torch.float64, device="cuda")

    def warp_path():
        tk = torch.zeros(1, dtype=torch.int64, device="cuda")
        xsum.lib().xsum_sum_segments_ws(x.data_ptr(), 0, keep, 0, offs_t.data_ptr(), out.data_ptr(), None, None, None,
                                        tk.data_ptr(), torch.cuda.current_stream().cuda_stream)
    ms_l = t_ms(lambda: xsum.sum_segments_csr(x, offs_t))
    ms_w = t_ms(warp_path)
    print(f"csr lengths U[0,{maxlen}]: {keep:9d} segments, {n} doubles: binding {ms_l * 1e3:9.1f} us "
          f"({n / ms_l / 1e6:6.1f} G/s) | warp per segment {ms_w * 1e3:9.1f} us ({n / ms_w / 1e6:6.1f} G/s)", flush=True)
