# Round-end measurement refresh (run on the GPU box from the repo root): GPU tests, smoke, every
# bench line, the reference arm, the c2 launch list and one ncu --set full capture of K2.
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/r_c2.json.log 2>&1
for c in c1 c3 c5 c5csr c2f32 c2f16 c2bf16 c2dim0 c5s16; do python bench.py --config $c --steps 100 > gpurun_out/r_$c.json.log 2>&1; done
python bench.py --config c4 --steps 20 > gpurun_out/r_c4.json.log 2>&1
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r_ref.json.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --sustained-s 0 > gpurun_out/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_accumulate -s 3 -c 1 -o gpurun_out/c2_final python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --sustained-s 0 > gpurun_out/ncu_f.log 2>&1
ls gpurun_out
