"""One named workload per call, for `ncu --set full -k regex:<kernel> -c 1` captures of the kernels
that are not the bench's dominant one (development tool).

    python tools/ncu_targets.py <target>

targets (kernel captured):
  seg_f32     binary32, 2^16 segments x 4096          (k_segments_small)
  seg_f16     binary16, 2^16 segments x 4096          (k_segments_h16)
  seg_bf16    bfloat16, 2^16 segments x 4096          (k_segments_h16)
  csr_lanes   ~2^27 doubles in 2^23 CSR rows of U[0, 32] (k_segments_lanes_csr)
  strided_split  [2^20, 256] doubles over dim 0       (k_sum_strided split + k_strided_merge)
  merge1024   merge of 1024 state images              (k_merge)
  finalize    finalize_round of a state               (k_finalize)
  sparse      to_sparse of a state, then a merge of 1024 sparse images (k_to_sparse, k_merge)
  c5csr       c5csr CSR segments (bench workload)     (k_segments)
  str_f64 / str_bf16 / str_f16 / str_f32  [4096, 65536] over dim 0 (K10s; k_sum_strided_h16 / _f32)
"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1605_05436_b200 as xsum  # noqa: E402
import synth  # noqa: E402


def main(t: str):
    xsum.build()
    synth.build()
    if t in ("seg_f32", "seg_f16", "seg_bf16"):
        x = synth.device_bits({"seg_f32": "c2f32", "seg_f16": "c2f16", "seg_bf16": "c2bf16"}[t])
        for _ in range(3):
            xsum.sum_segments(x, 4096)
    elif t == "csr_lanes":
        g = torch.Generator(device="cuda")
        g.manual_seed(5)
        lens = torch.randint(0, 33, (1 << 23,), device="cuda", generator=g)
        off = torch.zeros(lens.numel() + 1, dtype=torch.int64, device="cuda")
        off[1:] = torch.cumsum(lens, 0)
        x = synth.device_generate("c2", 0, int(off[-1].item()))
        for _ in range(3):
            xsum.sum_segments_csr(x, off)
    elif t == "strided_split":
        x = synth.device_generate("c2").view(1 << 20, 256)
        for _ in range(3):
            xsum.exact_sum_dim(x, 0)
    elif t == "str_f64":
        x = synth.device_generate("c2").view(4096, 65536)
        for _ in range(3):
            xsum.exact_sum_dim(x, 0)
    elif t in ("str_bf16", "str_f32", "str_f16"):
        x = synth.device_bits({"str_bf16": "c2bf16", "str_f32": "c2f32", "str_f16": "c2f16"}[t]).view(4096, 65536)
        for _ in range(3):
            xsum.exact_sum_dim(x, 0)
    elif t == "merge1024":
        x = synth.device_generate("c2", 0, 1 << 22)
        states = []
        for k in range(1024):
            a = xsum.Accumulator()
            a.add(x[k * 4096:(k + 1) * 4096])
            states.append(a.state.clone())
        st = torch.cat(states)
        m = xsum.Accumulator()
        for _ in range(3):
            m.reset().merge(st)
    elif t == "finalize":
        a = xsum.Accumulator().add(synth.device_generate("c2", 0, 1 << 20))
        for _ in range(3):
            a.finalize_async(canon=True)
    elif t == "sparse":
        x = synth.device_generate("c2", 0, 1 << 22)
        imgs, offs, pos = [], [], 0
        for k in range(1024):
            img, n = xsum.Accumulator().add(x[k * 4096:(k + 1) * 4096]).to_sparse()
            imgs.append(img.clone())
            offs.append(pos)
            pos += n
        images = torch.cat(imgs)
        offsets = torch.tensor(offs, dtype=torch.int64, device="cuda")
        m = xsum.Accumulator()
        for _ in range(3):
            m.reset().merge_sparse(images, offsets)
    elif t == "c5":
        x = synth.device_generate("c5")
        for _ in range(3):
            xsum.sum_segments(x, 4096)
    elif t == "c5csr":
        x = synth.device_generate("c5csr")
        off = synth.csr_offsets("c5csr", device="cuda")
        for _ in range(3):
            xsum.sum_segments_csr(x, off)
    else:
        raise SystemExit(f"unknown target {t}")
    torch.cuda.synchronize()
    print("ok", t)


if __name__ == "__main__":
    main(sys.argv[1])
