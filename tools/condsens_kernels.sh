#!/bin/bash
# per-kernel device times of one condition-number-sensitive sum (c3: every iteration runs) for each
# built variant of tools/variants.py (development tool; run on the GPU box)
for so in build/variants/libxsum_*.so; do
  echo "== $so"
  XSUM_DEV=1 XSUM_LIBRARY=$so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_cs|k_accumulate" --csv \
     python tools/condsens_run.py c3 1 2>/dev/null | grep gpu__time | awk -F'","' '{printf "%-50s %s %s\n", substr($5,1,50), $(NF), $(NF-1)}'
done
