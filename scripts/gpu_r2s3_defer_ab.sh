#!/bin/bash
# stores after all loads in the sparse phases (BBW_DEFER_ST=1) vs per-output load/store (0): config-5 bench, ab.py
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
lib() { echo paper_1808_08645_b200/native/$1/libbbwadg.so; }
for rep in 1 2; do
for v in ds0_74 ds1_74 c3_74; do
  BBWADG_LIB=$(lib $v) timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep --no-config4 \
    --elastic '' --two-d '' > gpurun_out/ds_bench_${v}_$rep.json 2> /dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/ds_bench_${v}_$rep.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
done
AB_REPS=2 timeout 900 python scripts/ab.py 5 3 ds0_53 ds1_53 c3_53 > gpurun_out/ds_ab.txt 2>&1
AB_REPS=2 timeout 900 python scripts/ab.py 7 4 ds0_74 ds1_74 c3_74 >> gpurun_out/ds_ab.txt 2>&1
cat gpurun_out/ds_ab.txt
