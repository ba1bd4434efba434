"""Exercise every libxsum entry point at small sizes (for compute-sanitizer runs).

    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1605_05436_b200 as xsum  # noqa: E402
import synth  # noqa: E402


def check(res, x):
    r, _ = oracle.exact_sum(x)
    assert res.bits == r.bits and res.flags == r.flags, (hex(res.bits), hex(r.bits))


def main():
    xsum.build()
    synth.build()
    x = synth.gen.generate("c4", 5, 300_001)
    x.view(np.uint64)[1234] = 0x7FF0000000000000
    buf = torch.empty(x.size + 2, dtype=torch.float64, device="cuda")
    for off in (0, 1):
        d = buf[off:off + x.size]
        d.copy_(torch.from_numpy(x))
        res, _ = xsum.exact_sum(d)
        check(res, x)
        acc = xsum.Accumulator().set_grid_limit(2)
        acc.add(d[:100_000]).add(d[100_000:])
        check(acc.result(), x)
    # float32
    f = synth.gen.generate("c1", 0, 70_003).astype(np.float32)
    fb = torch.empty(f.size + 4, dtype=torch.float32, device="cuda")
    for off in range(4):
        d = fb[off:off + f.size]
        d.copy_(torch.from_numpy(f))
        res, _ = xsum.exact_sum(d)
        check(res, f)
    # merge / states / host path
    a1 = xsum.Accumulator().add(buf[:1000])
    a2 = xsum.Accumulator().add(buf[1000:5000])
    tot = xsum.Accumulator().merge(torch.cat([a1.state, a2.state]))
    check(tot.result(), buf[:5000].cpu().numpy())
    h = xsum.Accumulator().add_host(x, stage_bytes=2 << 20)
    check(h.result(), x)
    # segments: general and streaming paths, CSR
    s = synth.gen.generate("c5", 0, 64 * 256)
    sd = torch.from_numpy(s).cuda()
    for seg_len, dd in ((256, sd), (255, sd[: 64 * 255]), (100, sd[1:6401])):
        vals, canon, flags = xsum.sum_segments(dd, seg_len, canon=True, flags=True)
        host = dd.cpu().numpy()
        for k in range(dd.numel() // seg_len):
            r, _ = oracle.exact_sum(host[k * seg_len:(k + 1) * seg_len])
            assert vals[k].item() == r.value
    offs = torch.tensor([0, 0, 3, 700, 701, 5000], dtype=torch.int64, device="cuda")
    vals, _, _ = xsum.sum_segments_csr(sd, offs, canon=True, flags=True)
    torch.cuda.synchronize()
    print("sanitize smoke ok, launches:", xsum.launch_count())


if __name__ == "__main__":
    main()
