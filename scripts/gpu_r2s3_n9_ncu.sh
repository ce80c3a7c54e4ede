#!/bin/bash
# ncu --set full of the config-3 stage kernel at (8,8) and (9,9) (n=44, 511,104 tets): occupancy and limiters
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for nm in "8 8" "9 9"; do
  set -- $nm
  timeout 900 ncu --set full --clock-control none -k regex:stage_kernel -s 5 -c 1 -o /tmp/c3_$1$2 \
    python bench.py --config 3 --N $1 --M $2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-sweep --no-config4 \
    --elastic '' --two-d '' > gpurun_out/c3_ncu_$1$2.log 2>&1
  ncu -i /tmp/c3_$1$2.ncu-rep --page raw --csv > gpurun_out/c3_raw_$1$2.csv 2>/dev/null
done
ls -la gpurun_out/c3_raw_*
