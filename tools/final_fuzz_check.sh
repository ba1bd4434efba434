#!/bin/bash
# Fuzzing (product and device-assert builds) and the GPU suite on the device-assert build after the
# k_merge leaf pipeline (GPU box; development tool). build/checked/libxsum.so: tools/checked_build.py.
mkdir -p gpurun_out
{ echo "product build, seeds 700000+:"; timeout 400 python tools/fuzz.py 240 700000 2>&1 | tail -3
  echo "checked build (XS_CHECKED device asserts), seeds 950000+:"; XSUM_DEV=1 XSUM_LIBRARY=build/checked/libxsum.so timeout 300 python tools/fuzz.py 150 950000 2>&1 | tail -3
} > gpurun_out/r02h_fuzz.txt; cat gpurun_out/r02h_fuzz.txt
XSUM_DEV=1 XSUM_LIBRARY=build/checked/libxsum.so timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02h_checked_suite.log 2>&1; echo "checked suite rc=$?"; tail -n 2 gpurun_out/r02h_checked_suite.log
