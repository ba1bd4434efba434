#!/bin/bash
# full GPU suite, the default bench line, its ncu launch list and the dominant kernel capture (GPU box; development tool)
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02_gpu_suite.log 2>&1; echo "suite rc=$?" 
tail -n 3 gpurun_out/r02_gpu_suite.log
timeout 900 python bench.py > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err; echo "bench rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c4_launches.csv python bench.py --steps 3 --warmup 3 > gpurun_out/r02_c4_launches.log 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_accumulate -c 1 -o gpurun_out/r02_c4_k_accumulate python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --sustained-s 0 > gpurun_out/r02_c4_ncu.log 2>&1; echo "ncu rc=$?"
