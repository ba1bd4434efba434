"""Run tools/op_bench.cu: warp-instructions per clock per SM for single integer ops."""
import ctypes
import os

import pynvml
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L = ctypes.CDLL(os.path.join(ROOT, "build", "libop_bench.so"))
L.op_bench.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
blocks, iters = 296, 4000
out = torch.empty(blocks * 1024, dtype=torch.int32, device="cuda")
names = ["add.u32 (IADD3)", "xor (LOP3)", "shf (SHF)", "mad.lo (IMAD)", "mad.hi (IMAD.HI)",
         "mad.wide+xor", "max.u32 (VIMNMX)", "setp+selp"]
for op, name in enumerate(names):
    st = torch.cuda.current_stream()
    L.op_bench(op, out.data_ptr(), blocks, 100, st.cuda_stream)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    L.op_bench(op, out.data_ptr(), blocks, iters, st.cuda_stream)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    warp_instr = blocks * 32 * iters * 8          # 32 warps/block x iters x 8 chains
    per_clk_sm = warp_instr / 148 / (ms * 1e-3 * mhz * 1e6)
    print(f"{name:20s} {ms:8.3f} ms  {per_clk_sm:5.2f} warp-instr/clk/SM @{mhz} MHz", flush=True)
