"""Sustained-load behaviour: kernel time per 100-launch window plus NVML power, clocks,
temperature and throttle reasons sampled alongside (development tool)."""
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402

import paper_1605_05436_b200 as xsum  # noqa: E402
import synth  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
x = synth.device_generate(sys.argv[1] if len(sys.argv) > 1 else "c2")
acc = xsum.Accumulator()
for _ in range(5):
    acc.sum(x)
torch.cuda.synchronize()
samples = []
stop = threading.Event()


def poll():
    while not stop.is_set():
        try:
            samples.append((time.perf_counter(), pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                            pynvml.nvmlDeviceGetTemperature(h, pynvml.NVML_TEMPERATURE_GPU),
                            pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        except Exception:
            pass
        time.sleep(0.02)


th = threading.Thread(target=poll, daemon=True)
t0 = time.perf_counter()
th.start()
W = 100
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(3000)]
for a, b in ev:
    a.record()
    acc.sum(x)
    b.record()
torch.cuda.synchronize()
stop.set()
th.join()
per = [a.elapsed_time(b) * 1e3 for a, b in ev]
for w in range(0, len(per), W * 3):
    print(f"launches {w:5d}-{w + W:5d}: median {statistics.median(per[w:w + W]):7.1f} us")
for s in samples[:: max(1, len(samples) // 25)]:
    print(f"t={s[0] - t0:6.3f}s power {s[1]:6.1f} W  sm {s[2]} MHz  mem {s[3]} MHz  temp {s[4]} C  reasons 0x{s[5]:x}")
