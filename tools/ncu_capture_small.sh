#!/bin/bash
# ncu --set full captures of the small helper kernels without one (GPU box; development tool):
# K12's k_cs_init / k_cs_exact_info / k_cs_final on c2, k_init_state, and the k_peer_selftest
# protocol kernel (virtual ranks in one cooperative launch).
mkdir -p gpurun_out
cap() {  # name regex skip cmd...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$rx" --launch-skip $skip -c 1 \
      -o gpurun_out/r02i_$name "$@" > gpurun_out/ncu_r02i_$name.log 2>&1 || echo "capture $name failed"
}
cap cs_init '^k_cs_init' 0 python tools/condsens_run.py c2 2
cap cs_exact_info '^k_cs_exact_info' 0 python tools/condsens_run.py c2 2
cap cs_final '^k_cs_final' 0 python tools/condsens_run.py c2 2
cap init_state '^k_init_state' 2 python tools/ncu_targets.py finalize
cap peer_selftest 'k_peer_selftest' 2 python tools/merge_run.py
ls gpurun_out/r02i_*
