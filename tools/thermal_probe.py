"""c2 throughput vs board state (development tool): batches of 200 back-to-back fused sums
(~75 ms each) under load, then idle gaps, logging GPU / HBM temperature, power, SM and memory
clocks and the clock-event reasons NVML reports."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml as nv  # noqa: E402
import torch  # noqa: E402

import paper_1605_05436_b200 as xsum  # noqa: E402
import synth  # noqa: E402

nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)


def state():
    t = nv.nvmlDeviceGetTemperature(h, nv.NVML_TEMPERATURE_GPU)
    try:
        mt = nv.nvmlDeviceGetFieldValues(h, [nv.NVML_FI_DEV_MEMORY_TEMP])[0].value.uiVal
    except Exception:
        mt = -1
    p = nv.nvmlDeviceGetPowerUsage(h) / 1000
    sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
    mem = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_MEM)
    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
    return f"gpu {t}C hbm {mt}C {p:.0f} W sm {sm} mem {mem} MHz reasons {r:#x}"


x = synth.device_generate("c2")
acc = xsum.Accumulator()
for _ in range(5):
    acc.sum(x)
torch.cuda.synchronize()


def batch(k=200):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        acc.sum(x)
    b.record()
    torch.cuda.synchronize()
    return x.numel() * k / (a.elapsed_time(b) * 1e6)


print("idle:", state(), flush=True)
for phase, (nb, gap) in enumerate([(30, 0.0), (5, 2.0), (5, 5.0), (3, 15.0)]):
    for i in range(nb):
        if gap:
            time.sleep(gap)
            s0 = state()
        else:
            s0 = ""
        g = batch()
        print(f"phase {phase} batch {i:2d} (gap {gap:4.1f} s): {g:6.1f} G/s   after: {state()}   before: {s0}",
              flush=True)
