"""Throughput of exact reductions over a non-last dimension (development tool): xsum_sum_strided
(K10, no transposing copy) vs the movedim + contiguous copy + segments path it replaced, with
torch.sum (not exact) for context. Event-timed medians."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1605_05436_b200 as xsum  # noqa: E402
import synth  # noqa: E402


def t_ms(f, reps=20):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        f()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


base = synth.device_generate("c2")                       # 2^28 doubles
for shape, dt in (((4096, 65536), torch.float64), ((65536, 4096), torch.float64), ((1 << 20, 256), torch.float64),
                  ((64, 4096, 1024), torch.float64), ((4096, 65536), torch.float32), ((4096, 65536), torch.bfloat16)):
    n = 1
    for s in shape:
        n *= s
    # narrow formats: the finite bit-pattern workloads (c2 doubles would overflow to Inf)
    x = {torch.float32: lambda: synth.device_bits("c2f32")[:n], torch.bfloat16: lambda: synth.device_bits("c2bf16")[:n],
         torch.float64: lambda: base[:n]}[dt]().reshape(shape)
    dim = 0 if len(shape) == 2 else 1
    nbytes = x.numel() * x.element_size()
    ms_new = t_ms(lambda: xsum.exact_sum_dim(x, dim))

    def old():
        xt = x.movedim(dim, -1).contiguous()
        return xsum._segments(xt.reshape(-1), xt.numel() // xt.shape[-1], xt.shape[-1], None, False, False)
    ms_old = t_ms(old)
    ms_torch = t_ms(lambda: torch.sum(x, dim))
    outer = 1
    for s in shape[:dim]:
        outer *= s
    inner = n // (outer * shape[dim])
    parts = xsum.lib().xsum_sum_strided_work_bytes(outer, shape[dim], inner, 0)
    print(f"{str(tuple(shape)):>20} {str(dt)[6:]:>8} dim {dim}: strided {ms_new * 1e3:8.1f} us "
          f"{nbytes / ms_new / 1e6:7.1f} GB/s (work {parts / 2**20:.1f} MiB) | movedim+segments {ms_old * 1e3:8.1f} us "
          f"| torch.sum (inexact) {ms_torch * 1e3:8.1f} us", flush=True)
