#!/bin/bash
# elastic kernel: unit-batches per work-queue ticket (BBWADG_ELASTIC_QCH = 1, 2, 4), elastic bench lines at n=56
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
for q in 1 2 4; do
  BBWADG_ELASTIC_QCH=$q timeout 900 python bench.py --n-cubes 8 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep \
    --no-config4 --two-d '' --elastic 7:2:f64,5:1:f64,9:2:f64 > gpurun_out/elqch_${q}_$rep.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/elqch_${q}_$rep.json').read().strip().splitlines()[-1]); e=d['elastic']
print('QCH=$q', {k: round(v['value']/1e10, 4) for k, v in e.items() if isinstance(v, dict) and 'value' in v})"
done
done
