#!/bin/bash
# diagnose the TMEM LSRK-state variant (BBW_LSRK_TMEM=1, tm74) against the default (d74): ab.py timing, then one
# ncu --set full capture of each at n=32 (196,608 tets), stall reasons and TMEM / L1 / occupancy metrics
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
AB_REPS=1 timeout 600 python scripts/ab.py 7 4 d74 tm74 > gpurun_out/tmem_ab.txt 2>&1
cat gpurun_out/tmem_ab.txt
for v in d74 tm74; do
  BBWADG_LIB=paper_1808_08645_b200/native/$v/libbbwadg.so timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:stage_kernel -s 5 -c 1 -o /tmp/tm_$v python bench.py --n-cubes 32 --steps 1 --warmup 1 --no-e2e \
    --no-cpu-baseline --no-sweep --no-config4 --elastic '' --two-d '' > gpurun_out/tmem_ncu_$v.log 2>&1
  ncu -i /tmp/tm_$v.ncu-rep --page raw --csv > gpurun_out/tmem_raw_$v.csv 2>/dev/null
  ncu -i /tmp/tm_$v.ncu-rep --page source --csv > gpurun_out/tmem_src_$v.csv 2>/dev/null
done
ls -la gpurun_out/tmem_*
