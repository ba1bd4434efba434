#!/bin/bash
# After the pipelined k_merge leaf loads (GPU box; development tool): the full GPU suite, smoke,
# merge latencies, and ncu --set full captures of k_merge on 1024 dense / sparse images.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02h_gpu_suite.log 2>&1; echo "suite rc=$?"; tail -n 2 gpurun_out/r02h_gpu_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02h_smoke.log
timeout 300 python tools/merge_run.py > gpurun_out/r02h_merge_run.txt 2>&1; echo "merge_run rc=$?"; cat gpurun_out/r02h_merge_run.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_merge --launch-skip 1 -c 1 -o gpurun_out/r02h_merge1024 python tools/ncu_targets.py merge1024 > gpurun_out/ncu_r02h_1.log 2>&1; echo "ncu1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_merge --launch-skip 1 -c 1 -o gpurun_out/r02h_merge_sparse python tools/ncu_targets.py sparse > gpurun_out/ncu_r02h_2.log 2>&1; echo "ncu2 rc=$?"
