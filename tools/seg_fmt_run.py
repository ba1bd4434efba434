"""Time segmented sums per input format (development tool): 2^28 elements of the c2f32 / c2f16 /
c2bf16 workloads (or c2 for binary64) in equal segments of 4096, CSR of the same bounds, and the
ragged CSR bounds of c5csr (lengths 1..8192)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1605_05436_b200 as xsum  # noqa: E402
import synth  # noqa: E402

for name in ("c2", "c2f32", "c2f16", "c2bf16"):
    x = synth.device_generate("c2") if name == "c2" else synth.device_bits(name)
    L = 4096
    offs = torch.arange(0, x.numel() + 1, L, dtype=torch.int64, device="cuda")
    ragged = synth.csr_offsets("c5csr", device="cuda")
    for kind in ("equal", "csr", "ragged"):
        f = {"equal": lambda: xsum.sum_segments(x, L), "csr": lambda: xsum.sum_segments_csr(x, offs),
             "ragged": lambda: xsum.sum_segments_csr(x, ragged)}[kind]
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            f()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 20
        n = x.numel() if kind != "ragged" else int(ragged[-1].item())
        print(f"{name:7s} {kind:6s}: {ms * 1e3:8.1f} us  {n / ms / 1e6:7.1f} G elem/s  "
              f"{n * x.element_size() / ms / 1e6:7.1f} GB/s", flush=True)
