"""Run a few fused sums of one input dtype (development / ncu target).

    python tools/dtype_run.py {f64,f32,f16,bf16} [n_log2=30] [reps=5]
"""
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_1605_05436_b200 as xsum  # noqa: E402


def data(kind: str, n: int):
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    if kind in ("f16", "bf16"):
        x = torch.randint(-32768, 32767, (n,), dtype=torch.int16, device="cuda", generator=g)
        em = 0x7C00 if kind == "f16" else 0x7F80
        return torch.where((x & em) == em, x ^ 0x400, x).view(torch.float16 if kind == "f16" else torch.bfloat16)
    if kind == "f32":
        x = torch.randint(-2 ** 31, 2 ** 31 - 1, (n,), dtype=torch.int32, device="cuda", generator=g)
        return torch.where((x & 0x7F800000) == 0x7F800000, x ^ 0x800000, x).view(torch.float32)
    x = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    return x


if __name__ == "__main__":
    kind = sys.argv[1]
    n = 1 << int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 30
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    x = data(kind, n)
    acc = xsum.Accumulator()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record()
        acc.sum(x)
        b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)[reps // 2]
    print(f"{kind} n={n} median {ms:.3f} ms  {n / ms / 1e6:.1f} G elem/s  {x.element_size() * n / ms / 1e6:.1f} GB/s")
