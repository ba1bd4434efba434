#!/bin/bash
# ncu --set full captures of the kernels changed late in round 2 (K12 tree kernels, K11s) (GPU box;
# development tool). On c3 the k_cs_tree launches are <2,1>, <2,0>, <2,0>, <4,1>, ...
set -u
cap() {  # name regex skip cmd...
  local name=$1 rx=$2 skip=$3; shift 3
  ncu --set full --clock-control none --import-source on -k regex:"$rx" --launch-skip $skip -c 1 \
      -o gpurun_out/r02_$name "$@" > gpurun_out/ncu_$name.log 2>&1 || echo "capture $name failed"
}
cap c3cs_k_cs_tree2 '^k_cs_tree$' 0 python tools/condsens_run.py c3 1
cap c3cs_k_cs_tree4 '^k_cs_tree$' 3 python tools/condsens_run.py c3 1
ls -la gpurun_out/*.ncu-rep
