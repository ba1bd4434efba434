"""Run tools/smem_bench.cu modes; prints summands per clock per SM for each RMW form."""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L = ctypes.CDLL(os.path.join(ROOT, "build", "libsmem_bench.so"))
L.smem_bench.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
import pynvml  # noqa: E402
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
out = torch.empty(148 * 512, dtype=torch.int64, device="cuda")
iters = 2000
import sys as _sys
MODES = [(0, "LDS+add+STS (64-bit)"), (1, "atomicAdd shared u64"), (2, "red.shared.add.u64"),
         (3, "red.shared.add.u32"), (4, "STS.64 only (random digit)"), (5, "LDS.64 only (random digit)"),
         (6, "RMW same digit all lanes")]
sel = [int(a) for a in _sys.argv[1:]]
for mode, name in [m for m in MODES if not sel or m[0] in sel]:
    st = torch.cuda.current_stream()
    for _ in range(2):
        L.smem_bench(mode, out.data_ptr(), 148, iters, st.cuda_stream)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    rc = L.smem_bench(mode, out.data_ptr(), 148, iters, st.cuda_stream)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    summands = 148 * 512 * iters * 8
    per_clk_sm = summands / 148 / (ms * 1e-3 * mhz * 1e6)
    print(f"{name:24s} rc={rc} {ms:8.3f} ms  {summands / ms / 1e6:8.1f} G summands/s  {per_clk_sm:.2f} /clk/SM @{mhz} MHz")
