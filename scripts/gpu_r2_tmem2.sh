#!/bin/bash
# TMEM LSRK-state variant with the grid forced to 4 CTAs per SM (the occupancy query returns 1 for it)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python - <<'PY' > gpurun_out/tmem_occ.txt 2>&1
import ctypes, os
for v in ["d74", "tm74"]:
    os.environ["BBWADG_LIB"] = f"paper_1808_08645_b200/native/{v}/libbbwadg.so"
PY
AB_REPS=2 timeout 600 python scripts/ab.py 7 4 d74 tm74 > gpurun_out/tmem_ab2.txt 2>&1
BBWADG_FORCE_BLOCKS_PER_SM=4 AB_REPS=2 timeout 600 python scripts/ab.py 7 4 d74 tm74 >> gpurun_out/tmem_ab2.txt 2>&1
cat gpurun_out/tmem_ab2.txt
BBWADG_FORCE_BLOCKS_PER_SM=4 BBWADG_LIB=paper_1808_08645_b200/native/tm74/libbbwadg.so timeout 900 ncu --metrics \
  gpu__time_duration.sum,sm__warps_active.avg.per_cycle_active,launch__grid_size,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed \
  --clock-control none -k regex:stage_kernel -s 5 -c 1 --csv python bench.py --n-cubes 32 --steps 1 --warmup 1 --no-e2e \
  --no-cpu-baseline --no-sweep --no-config4 --elastic '' --two-d '' 2>&1 | grep -E "duration|warps_active|grid_size|wavefronts"
