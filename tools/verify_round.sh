mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02v_gpu_suite.log 2>&1; echo "suite rc=$?"
tail -n 3 gpurun_out/r02v_gpu_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02v_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02v_smoke.log
timeout 900 python bench.py > gpurun_out/r02v_bench.json 2> gpurun_out/r02v_bench.err; echo "bench rc=$?"; cat gpurun_out/r02v_bench.json | head -c 3000
timeout 600 python bench.py --impl reference > gpurun_out/r02v_ref.json 2> gpurun_out/r02v_ref.err; echo "ref rc=$?"; head -c 1500 gpurun_out/r02v_ref.json
