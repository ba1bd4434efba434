#!/bin/bash
# every bench workload once (GPU box): JSON lines to gpurun_out/r02_bench_<cfg>.json (development tool)
for c in c4 c2 c1 c3 c5 c5csr c5s16 c2f32 c2f16 c2bf16 c2dim0 c2cs c3cs; do
  steps=20; [ "$c" = c3cs ] && steps=5; [ "$c" = c2cs ] && steps=10
  timeout 900 python bench.py --config $c --steps $steps --warmup 5 > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err
  echo "$c rc=$?"
done
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r02_bench_reference.json 2>&1
