"""c5csr timing by method (development tool): per-step events vs the span of back-to-back calls, and the host enqueue cost per call."""
import sys, os, statistics
sys.path.insert(0, os.getcwd())
import torch, synth, paper_1605_05436_b200 as xsum
x = synth.device_generate("c5csr"); csr = synth.csr_offsets("c5csr", device="cuda")
for _ in range(5): xsum.sum_segments_csr(x, csr)
torch.cuda.synchronize()
K = 50
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
for a, b in ev:
    a.record(); xsum.sum_segments_csr(x, csr); b.record()
torch.cuda.synchronize()
t = [a.elapsed_time(b) * 1e3 for a, b in ev]
print("per-step median %.1f mean %.1f min %.1f max %.1f" % (statistics.median(t), statistics.mean(t), min(t), max(t)))
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(K): xsum.sum_segments_csr(x, csr)
b.record(); torch.cuda.synchronize()
print("span/K %.1f" % (a.elapsed_time(b) * 1e3 / K))
import time
t0 = time.perf_counter()
for _ in range(K): xsum.sum_segments_csr(x, csr)
t1 = time.perf_counter(); torch.cuda.synchronize()
print("host enqueue per call %.1f us" % ((t1 - t0) / K * 1e6))
