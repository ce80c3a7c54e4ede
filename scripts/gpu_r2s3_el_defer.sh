#!/bin/bash
# elastic (7,2) with and without the store deferral of the shared sparse phases (face_sum3, sum4, upward sweep)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
for v in e72d0 e72d1; do
  BBWADG_LIB=paper_1808_08645_b200/native/$v/libbbwadg.so timeout 900 python bench.py --config 4 --N 7 --M 2 --n-cubes 8 \
    --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep --no-config4 --two-d '' --elastic 7:2:f64 \
    > gpurun_out/eld_${v}_$rep.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/eld_${v}_$rep.json').read().strip().splitlines()[-1]); e=d['elastic']['N7M2f64']; print('$v', e['value'], e['ms_per_step'])"
done
done
