"""Sustained back-to-back runs (~3 s each) of (a) the exact sum K2 over c2 and (b) a pure read
of the same 2 GiB (synth's streaming probe, no accumulation), with NVML power / SM clock / throttle
reasons: is the 1000 W cap reached by the HBM stream or by the SM work? (development tool)"""
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
x = synth.device_generate("c2")
nbytes = x.numel() * 8
acc = xsum.Accumulator()
lib = synth.cuda_lib()
blocks = 2 * torch.cuda.get_device_properties(0).multi_processor_count
out = torch.empty(blocks * 512, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream()


def run(name, fn, seconds=3.0):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    samples, stop = [], threading.Event()

    def poll():
        while not stop.is_set():
            try:
                samples.append((pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                                pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
            except Exception:
                pass
            time.sleep(0.02)
    th = threading.Thread(target=poll, daemon=True)
    th.start()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = 0
    a.record()
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        for _ in range(50):
            fn()
        k += 50
        torch.cuda.synchronize()
    b.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = a.elapsed_time(b) / k
    late = samples[len(samples) // 2:]
    print(f"{name:12s} {nbytes / ms / 1e6:7.0f} GB/s sustained  ({ms * 1e3:.0f} us per pass, {k} passes)  "
          f"power median {statistics.median(p for p, _, _ in late):.0f} W  SM {statistics.median(c for _, c, _ in late):.0f} MHz  "
          f"reasons {sorted({hex(r) for _, _, r in late})}")


run("exact sum K2", lambda: acc.sum(x))
run("read probe", lambda: lib.synth_probe_read(x.data_ptr(), nbytes, out.data_ptr(), 1, blocks, 512, st.cuda_stream))
time.sleep(5)
run("exact sum K2", lambda: acc.sum(x))
