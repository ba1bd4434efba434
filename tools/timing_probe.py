"""Where the fixed cost of a fused sum goes: an XS_TIMING=1 build of libxsum stamps %globaltimer
per block (start, stream done, warp combines done, arrival atomic returned) and in the last block
(grid sum read, rounded) into a scratch area of timing builds; this prints the spread (development
tool).

    python tools/timing_probe.py build     # here
    python tools/timing_probe.py run       # GPU box
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SO = os.path.join(ROOT, "build", "timing", "libxsum.so")

if sys.argv[1] == "build":
    from paper_1605_05436_b200 import _build as b
    os.makedirs(os.path.dirname(SO), exist_ok=True)
    subprocess.check_call(["nvcc", *b.ARCH, *b.FLAGS, "-DXS_TIMING=1", "-I", b.INCLUDE, "-shared", "-o", SO,
                           *b.sources()])
    print(SO)
    sys.exit(0)

os.environ["XSUM_DEV"] = "1"
os.environ["XSUM_LIBRARY"] = SO
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1605_05436_b200 as xsum  # noqa: E402
import synth  # noqa: E402

D, MAXB = 42, 1024
acc = xsum.Accumulator()
for k in (10, 20, 28):
    x = synth.device_generate("c2")[: 1 << k].clone()
    for _ in range(3):
        acc.sum(x)
    torch.cuda.synchronize()
    acc.scratch.zero_()
    acc.sum(x)
    torch.cuda.synchronize()
    stamps = acc.scratch[1024:1024 + 8 * 6 * MAXB].view(torch.int64).cpu().numpy().reshape(6, MAXB)
    st = {j: stamps[j] for j in range(6)}
    nb = int((st[0] != 0).sum())
    t0 = st[0][:nb].min()
    rel = {j: (st[j][:nb] - t0) / 1e3 for j in range(4)}
    print(f"n=2^{k} blocks={nb}: start {rel[0].min():.2f}..{rel[0].max():.2f} us, stream done "
          f"{rel[1].min():.2f}..{rel[1].max():.2f}, combines done {rel[2].min():.2f}..{rel[2].max():.2f}, "
          f"arrival {rel[3].min():.2f}..{rel[3].max():.2f}; last block merged {(st[4][0] - t0) / 1e3:.2f}, "
          f"rounded {(st[5][0] - t0) / 1e3:.2f} us")
