#!/bin/bash
# DEFER_ST=2 (also C1's r_p and B2's gradient stores after their loads) vs the default DEFER_ST=1, config-5 bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
for v in default d2_74; do
  if [ $v = default ]; then lib=paper_1808_08645_b200/native/libbbwadg.so; else lib=paper_1808_08645_b200/native/$v/libbbwadg.so; fi
  BBWADG_LIB=$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep --no-config4 \
    --elastic '' --two-d '' > gpurun_out/d2_bench_${v}_$rep.json 2> /dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/d2_bench_${v}_$rep.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
done
