#!/bin/bash
# packed reduction table (BBW_RED32: 4 B per output) vs ushort4 (8 B): config-5 bench and ab.py (5,3)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
lib() { echo paper_1808_08645_b200/native/$1/libbbwadg.so; }
for rep in 1 2; do
for v in r16_74 r32_74; do
  BBWADG_LIB=$(lib $v) timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep --no-config4 \
    --elastic '' --two-d '' > gpurun_out/red_bench_${v}_$rep.json 2> /dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/red_bench_${v}_$rep.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
done
AB_REPS=2 timeout 900 python scripts/ab.py 5 3 r16_53 r32_53 > gpurun_out/red_ab.txt 2>&1
AB_REPS=2 timeout 900 python scripts/ab.py 7 4 r16_74 r32_74 >> gpurun_out/red_ab.txt 2>&1
cat gpurun_out/red_ab.txt
