#!/bin/bash
# elastic: remaining GPU tests, bench lines, ncu launch list + one full capture of the elastic kernel
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 900 python -m pytest tests/test_gpu_elastic.py -q -k "rate or mu_zero or validates" 2>&1 | tail -5 ) > gpurun_out/el_tests2.txt
timeout 900 python bench.py --steps 3 --warmup 3 --no-sweep --no-config4 --no-cpu-baseline --no-e2e > gpurun_out/bench_el.json 2> gpurun_out/bench_el.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:elastic_stage -s 3 -c 1 -o gpurun_out/prof_el72 \
  python bench.py --steps 1 --warmup 1 --no-sweep --no-config4 --no-cpu-baseline --no-e2e --elastic 7:2:f64 --elastic-n 24 --n-cubes 16 > gpurun_out/ncu_el.log 2>&1
ncu -i gpurun_out/prof_el72.ncu-rep --page raw --csv > gpurun_out/el72_raw.csv 2>/dev/null
