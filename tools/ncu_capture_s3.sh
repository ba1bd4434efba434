#!/bin/bash
# ncu --set full captures of the kernels changed late in round 2 (GPU box; summarise with tools/ncu_summary.py)
set -u
mkdir -p gpurun_out
cap() {   # name target kernel-regex
  ncu --set full --clock-control none --import-source on -k regex:"$3" -c 1 -o gpurun_out/r02s_$1 \
      python tools/ncu_targets.py $2 > gpurun_out/ncu_s3_$1.log 2>&1 || echo "capture $1 failed"
}
cap c5 c5 k_segments_halfz
cap c5csr c5csr "^k_segments$"
cap str_f64 str_f64 k_sum_strided_sk
cap str_f32 str_f32 k_sum_strided_f32_sk
cap str_bf16 str_bf16 k_sum_strided_h16_sk
cap seg_f32 seg_f32 k_segments_smallq
cap seg_bf16 seg_bf16 k_segments_h16q
ls gpurun_out/r02s_*.ncu-rep
