mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "sparse or merge" > gpurun_out/r02g_sparse_tests.log 2>&1; echo "tests rc=$?"; tail -n 3 gpurun_out/r02g_sparse_tests.log
timeout 300 python tools/merge_run.py > gpurun_out/r02g_merge_run.txt 2>&1; echo "merge_run rc=$?"; tail -20 gpurun_out/r02g_merge_run.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_merge --launch-skip 1 -c 1 -o gpurun_out/r02g_merge_sparse python tools/ncu_targets.py sparse > gpurun_out/ncu_r02g.log 2>&1; echo "ncu rc=$?"
