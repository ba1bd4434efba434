"""Build libxsum.so in-tree for sm_100a (nvcc; no torch extension machinery)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
SO = os.path.join(HERE, "libxsum.so")
SOURCES = ["api.cu", "accumulate.cu", "accumulate_h16.cu", "accumulate_f32.cu", "merge_finalize.cu", "segments.cu", "segments_small.cu", "strided.cu", "segments_lanes.cu", "segments_half.cu", "condsens.cu"]
HEADERS = ["band_round.cuh", "xsum_device.cuh", "xsum_kernels.h", "grid_tail.cuh", "h16_common.cuh", "lane_round.cuh",
           "f32_bins.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr"]


def sources() -> list[str]:
    return [os.path.join(CSRC, s) for s in SOURCES]


def deps() -> list[str]:
    return sources() + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "xsum.h"),
                                                                   os.path.abspath(__file__)]


def stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(d) > t for d in deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return SO
    cmd = ["nvcc", *ARCH, *FLAGS, "-I", INCLUDE, "-shared", "-o", SO, *sources()]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(SO)
