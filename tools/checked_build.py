"""Build libxsum with device asserts (XS_CHECKED=1) into build/checked/, for running the GPU
test-suite as a bounds / int64-headroom check:

    python tools/checked_build.py && XSUM_DEV=1 XSUM_LIBRARY=build/checked/libxsum.so pytest tests -m gpu
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1605_05436_b200 import _build as b  # noqa: E402

out = os.path.join(ROOT, "build", "checked")
os.makedirs(out, exist_ok=True)
so = os.path.join(out, "libxsum.so")
subprocess.check_call(["nvcc", *b.ARCH, *b.FLAGS, "-DXS_CHECKED=1", "-I", b.INCLUDE, "-shared", "-o", so,
                       *b.sources()])
print(so)
