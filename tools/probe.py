"""Read-bandwidth probe sweep over the c2 input (2 GiB): one line per (variant, blocks, threads)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402

x = synth.device_generate("c2")
names = {0: "tiles U4 L2::256B", 1: "tiles U8 L2::256B", 2: "tiles U4 nohint", 3: "tiles U4 .cs",
         4: "chunks U4", 5: "chunks U8", 6: "tiles U16"}
for variant, blocks, threads in [(0, 148, 512), (1, 148, 512), (6, 148, 512), (2, 148, 512), (3, 148, 512),
                                 (0, 296, 512), (0, 592, 512), (1, 296, 512), (0, 1184, 256), (1, 592, 512),
                                 (4, 148, 512), (5, 148, 512), (5, 592, 512), (1, 148, 1024), (6, 296, 512)]:
    g = synth.probe_read_gbs(x, variant, blocks, threads)
    print(f"{names[variant]:22s} blocks={blocks:5d} threads={threads:4d}  {g:8.1f} GB/s", flush=True)
