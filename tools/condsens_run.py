"""Run the condition-number-sensitive sum (K12) on a config once per call, for ncu / timing
(development tool).   python tools/condsens_run.py [c2|c3] [reps]"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1605_05436_b200 as xsum  # noqa: E402
import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
x = synth.device_generate(cfg)
work = torch.empty(xsum.condsens_work_bytes(x.numel()), dtype=torch.uint8, device="cuda")
for _ in range(reps):
    res, info, _ = xsum.sum_condsens(x, 1, work=work)
torch.cuda.synchronize()
print(xsum.CondSensInfo.from_bytes(info.cpu().numpy().tobytes()))
