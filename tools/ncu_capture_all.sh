#!/bin/bash
# ncu --set full captures of the non-dominant kernels (tools/ncu_targets.py), one report each under
# gpurun_out/ (run on the GPU box; summarise with tools/ncu_summary.py)
set -u
cap() {   # target kernel-regex
  ncu --set full --clock-control none --import-source on -k regex:"$2" -c 1 -o gpurun_out/r02_$1 \
      python tools/ncu_targets.py $1 > gpurun_out/ncu_$1.log 2>&1 || echo "capture $1 failed"
}
cap seg_f32 k_segments_small
cap seg_f16 k_segments_h16
cap seg_bf16 k_segments_h16
cap csr_lanes k_segments_lanes_csr
cap strided_split k_sum_strided
cap merge1024 k_merge
cap finalize k_finalize
cap c5csr "k_segments[^_]"
ncu --set full --clock-control none --import-source on -k regex:k_strided_merge -c 1 -o gpurun_out/r02_strided_merge \
    python tools/ncu_targets.py strided_split > gpurun_out/ncu_strided_merge.log 2>&1 || echo "capture strided_merge failed"
ls gpurun_out/r02_*.ncu-rep
