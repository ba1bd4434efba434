"""Build and time compile-time variants of the accumulate kernel (development tool).

    python tools/variants.py build [name ...]   # here (nvcc cross-compiles)
    python tools/variants.py run [cfg ...]      # on the GPU box: one JSON line per built variant
cfg: c1..c5 (binary64 configs), c5seg (segments of c5), c5csr (CSR segments), f32 / f16 / bf16 (random finite
patterns), n<k> (the first 2^k elements of c2).
Variants named exp* are diagnostic builds that compute WRONG sums (timing only)."""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "build", "variants")
# name -> extra nvcc defines
VARIANTS = {
    "product": [],
    "base": [],        # build this one from another checkout of the sources for same-box A/B
    # examples of compile-time knobs (see the kernels): register-buffer depth of each kernel
    "acc_nb4": ["-DXS_ACC_NB=4"],
    "acc_nb3": ["-DXS_ACC_NB=3"],
    "acc_u2nb8": ["-DXS_ACC_U=2", "-DXS_ACC_NB=8"],
    "acc_w12": ["-DXS_ACC_WARPS=12"],
    "seg_nb4": ["-DXS_SEG_NB=4"],
    "seg_u2nb4": ["-DXS_SEG_U=2", "-DXS_SEG_NB=4"],
    "seg_u2nb8": ["-DXS_SEG_U=2", "-DXS_SEG_NB=8"],
    "seg_u1nb8": ["-DXS_SEG_U=1", "-DXS_SEG_NB=8"],
    "seg_u1nb16": ["-DXS_SEG_U=1", "-DXS_SEG_NB=16"],
    "lanes0": ["-DXS_SEG_LANES_MAX=0"],
    "seg_whole": ["-DXS_SEG_HALF=0"],
    "sh_q8u4": ["-DXS_SH_LPS=8", "-DXS_SH_U=4"],
    "sh_u4nb4": ["-DXS_SH_U=4", "-DXS_SH_NB=4"],
    "sh_u4nb3": ["-DXS_SH_U=4", "-DXS_SH_NB=3"],
    "sh_u8nb3": ["-DXS_SH_U=8", "-DXS_SH_NB=3"],
    "sh_u2nb8": ["-DXS_SH_U=2", "-DXS_SH_NB=8"],
    "sl_full": ["-DXS_SL_FULL"],
    "slfast0": ["-DXS_SL_FAST=0"],
    "slnb2": ["-DXS_SLS_NBUF=2"],
    "slnb2fast0": ["-DXS_SLS_NBUF=2", "-DXS_SL_FAST=0"],
    "cs2g5": ["-DXS_CS2_G=5"],
    "cs4g4": ["-DXS_CS4_G=4"],
    "cs4g4m2": ["-DXS_CS4_G=4", "-DXS_CS4_MINB=2"],
    "cs4g5": ["-DXS_CS4_G=5"],
    "csslots4": ["-DXS_CS_SLOTS=4"],
    "csslots2": ["-DXS_CS_SLOTS=2"],
    "cs2g5_4g4m2": ["-DXS_CS2_G=5", "-DXS_CS4_G=4", "-DXS_CS4_MINB=2"],
    "cs2g6_4g4m2": ["-DXS_CS2_G=6", "-DXS_CS4_G=4", "-DXS_CS4_MINB=2"],
    "cs2g5_4g5m2": ["-DXS_CS2_G=5", "-DXS_CS4_G=5", "-DXS_CS4_MINB=2"],
    "sl_nopf": ["-DXS_SL_PF=0"],
    "sl_notma": ["-DXS_SL_TMA=0"],
    "sls_nbuf2": ["-DXS_SLS_NBUF=2"],
    "h16q0": ["-DXS_H16Q=0"],
    "hq_lps4": ["-DXS_HQ_LPS=4"],
    "str_nb3": ["-DXS_STR_NB=3"],
    "strh0": ["-DXS_STRH=0"],
    "strh_unr8": ["-DXS_STRH_UNR=8"],
    "str_nb6": ["-DXS_STR_NB=6"],
    "str_u4nb8": ["-DXS_STR_UNR=4", "-DXS_STR_NB=8"],
    "exp_seg_noepi": ["-DXS_EXP_SEG_NOEPI"],
    "exp_seg_noacc": ["-DXS_EXP_SEG_NOACC"],
    "h16_nb2": ["-DXS_H16_NB=2"],
    "h16_ldsts": ["-DXS_H16_LDSTS"],
    "f32b_nb4": ["-DXS_F32B_NB=4"],
    "sz0": ["-DXS_SH_Z=0"],
    "sz_u4nb4": ["-DXS_SZ_U=4", "-DXS_SZ_NB=4"],
    "sz_u2nb8": ["-DXS_SZ_U=2", "-DXS_SZ_NB=8"],
    "sz_coh": ["-DXS_SZ_COH=1"],
    "sz_w8": ["-DXS_SZ_WARPS=8", "-DXS_SZ_MINB=2"],
    "strsk0": ["-DXS_STR_SK=0"],
    "segc_w16": ["-DXS_SEGC_WARPS=16", "-DXS_SEGC_MINB=1"],
    "sseg_w16": ["-DXS_SSEG_WARPS=16", "-DXS_SSEG_MINB=1"],
    "segc_nb3": ["-DXS_SEGC_NB=3"],
    "segu_w16": ["-DXS_SEGU_WARPS=16", "-DXS_SEGU_MINB=1"],
    "exp_sz_noepi": ["-DXS_EXP_SZ_NOEPI"],
}


def build(names=None):
    from paper_1605_05436_b200 import _build as b
    os.makedirs(OUT, exist_ok=True)
    for name, defs in VARIANTS.items():
        if names and name not in names:
            continue
        so = os.path.join(OUT, f"libxsum_{name}.so")
        cmd = ["nvcc", *b.ARCH, *b.FLAGS, *defs, "-I", b.INCLUDE, "-shared", "-o", so, *b.sources()]
        subprocess.check_call(cmd)
        print(so)


def run_one(so: str, cfg: str, steps: int):
    code = f"""
import os, sys, json, statistics
sys.path.insert(0, {ROOT!r})
os.environ["XSUM_DEV"] = "1"
os.environ["XSUM_LIBRARY"] = {so!r}
import torch, synth, paper_1605_05436_b200 as xsum
if {cfg!r}.startswith("n"):
    x = synth.device_generate("c2")[: 1 << int({cfg!r}[1:])].clone()
elif {cfg!r} == "f32":
    g = torch.Generator(device="cuda"); g.manual_seed(1)
    x = torch.randint(-2 ** 31, 2 ** 31 - 1, (1 << 29,), dtype=torch.int32, device="cuda", generator=g)
    x = torch.where((x & 0x7F800000) == 0x7F800000, x ^ 0x800000, x).view(torch.float32)
elif {cfg!r} in ("f16", "bf16"):
    g = torch.Generator(device="cuda"); g.manual_seed(1)
    x = torch.randint(-32768, 32767, (1 << 30,), dtype=torch.int16, device="cuda", generator=g)
    em = 0x7C00 if {cfg!r} == "f16" else 0x7F80
    x = torch.where((x & em) == em, x ^ 0x400, x).view(torch.float16 if {cfg!r} == "f16" else torch.bfloat16)
elif {cfg!r}.startswith("str"):
    base = synth.device_generate("c2")
    shp = {{"str64": (4096, 65536), "str1m": (1 << 20, 256), "str3d": (64, 4096, 1024)}}.get({cfg!r}, (4096, 65536))
    x = base.reshape(shp)
    if {cfg!r} in ("strbf16", "strf16", "strf32"):
        x = synth.device_bits({{"strbf16": "c2bf16", "strf16": "c2f16", "strf32": "c2f32"}}[{cfg!r}]).reshape(shp)
    class _D:
        def sum(self, x):
            global seg_v
            seg_v = xsum.exact_sum_dim(x, 1 if x.dim() == 3 else 0)
            return xsum_res, None
    xsum_res = xsum.Accumulator().sum(base[:1024])[0]
elif {cfg!r} in ("cs2", "cs3"):
    x = synth.device_generate("c2" if {cfg!r} == "cs2" else "c3")
    class _K:
        def sum(self, x):
            r, _, _ = xsum.sum_condsens(x, 1)
            return r, None
elif {cfg!r} == "c5csr":
    x = synth.device_generate("c5csr")
    csr = synth.csr_offsets("c5csr", device="cuda")
elif {cfg!r} == "csrl32":                       # sparse-matrix-like rows: U[0, 32] doubles (K11c)
    g = torch.Generator(device="cuda"); g.manual_seed(5)
    lens = torch.randint(0, 33, (1 << 23,), device="cuda", generator=g)
    csr = torch.zeros(lens.numel() + 1, dtype=torch.int64, device="cuda")
    csr[1:] = torch.cumsum(lens, 0)
    x = synth.device_generate("c2", 0, int(csr[-1].item()))
elif {cfg!r} in ("f16seg", "bf16seg", "f32seg"):
    pass
elif {cfg!r} in ("c2s64", "c2s256", "c2s64k", "c2s768"):
    x = synth.device_generate("c2")
    x = x[: x.numel() // 768 * 768] if {cfg!r} == "c2s768" else x
else:
    x = synth.device_generate({cfg!r}.replace("seg", ""))
acc = _D() if {cfg!r}.startswith("str") else _K() if {cfg!r} in ("cs2", "cs3") else xsum.Accumulator()
if {cfg!r} in ("c5csr", "csrl32"):
    class _C:
        def sum(self, x):
            global seg_v
            seg_v, _, _ = xsum.sum_segments_csr(x, csr)
            return xsum_res, None
    xsum_res = acc.sum(x)[0]
    acc = _C()
if {cfg!r} in ("f16seg", "bf16seg", "f32seg"):
    x = synth.device_bits({{"f16seg": "c2f16", "bf16seg": "c2bf16", "f32seg": "c2f32"}}[{cfg!r}])
if {cfg!r}.endswith("seg") or {cfg!r} in ("c5s16", "c2s64", "c2s256", "c2s64k", "c2s768"):
    SEGL = {{"c5s16": 16, "c2s64": 64, "c2s256": 256, "c2s64k": 65536, "c2s768": 768}}.get({cfg!r}, 4096)
    class _S:
        def sum(self, x):
            global seg_v
            seg_v, _, _ = xsum.sum_segments(x, SEGL)
            return xsum_res, None
    xsum_res = acc.sum(x)[0]
    acc = _S()
for _ in range(5): acc.sum(x)
torch.cuda.synchronize()
import time as _t
_t0 = _t.perf_counter()
while _t.perf_counter() - _t0 < float(os.environ.get("VARIANT_SUSTAIN", "0")):   # power-capped steady state
    for _ in range(20): acc.sum(x)
    torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range({steps})]
for a, b in ev:
    a.record(); acc.sum(x); b.record()
torch.cuda.synchronize()
ms = statistics.median(a.elapsed_time(b) for a, b in ev)
res, _ = acc.sum(x); r = xsum.Result.from_bytes(res.cpu().numpy().tobytes())
import hashlib
check = hashlib.sha256(seg_v.cpu().numpy().tobytes()).hexdigest()[:16] if {cfg!r}.endswith(("seg", "csr", "s16", "s64", "s256", "l32", "s64k", "s768")) or {cfg!r}.startswith("str") else hex(r.bits)
print(json.dumps(dict(so=os.path.basename({so!r}), cfg={cfg!r}, ms=ms, gdps=x.numel()/ms/1e6, gbs=x.element_size()*x.numel()/ms/1e6, check=check)))
"""
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    print(out.stdout.strip() or out.stderr[-2000:], flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    else:
        cfgs = sys.argv[2:] or ["c2"]
        reps = int(os.environ.get("VARIANT_REPS", "1"))
        for cfg in cfgs:
            for name in [v for _ in range(reps) for v in VARIANTS]:   # interleaved repetitions
                so = os.path.join(OUT, f"libxsum_{name}.so")
                if os.path.exists(so):
                    run_one(so, cfg, 50)
