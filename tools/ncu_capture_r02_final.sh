#!/bin/bash
# Round 2 last session (GPU box; development tool): parity of the segment-format kernels after the
# ping-pong register buffers in K9q / K9sq, their timings, ncu --set full captures of k_segments_h16q
# (bfloat16, binary16), k_segments_smallq (binary32), and k_to_sparse / k_merge on sparse images.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_segments_fmt.py tests/test_gpu_sparse.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02f_segfmt_tests.log 2>&1; echo "tests rc=$?"; tail -n 2 gpurun_out/r02f_segfmt_tests.log
timeout 600 python tools/seg_fmt_run.py > gpurun_out/r02f_seg_fmt_run.txt 2>&1; echo "seg_fmt rc=$?"; cat gpurun_out/r02f_seg_fmt_run.txt
cap() {  # name regex skip target
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$2" --launch-skip $3 -c 1 \
      -o gpurun_out/r02f_$1 python tools/ncu_targets.py $4 > gpurun_out/ncu_r02f_$1.log 2>&1 || echo "capture $1 failed"
}
cap seg_bf16 k_segments_h16q 1 seg_bf16
cap seg_f16 k_segments_h16q 1 seg_f16
cap seg_f32 k_segments_smallq 1 seg_f32
cap to_sparse k_to_sparse 100 sparse
cap merge_sparse k_merge 1 sparse
ls gpurun_out/r02f_*
