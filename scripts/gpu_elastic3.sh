#!/bin/bash
# elastic: full GPU parity after the layout change, bench lines, A/B of the register cap at (7,2)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 1500 python -m pytest tests/test_gpu_elastic.py -q -x 2>&1 | tail -5 ) > gpurun_out/el_tests3.txt
timeout 900 python bench.py --steps 2 --warmup 3 --no-sweep --no-config4 --no-cpu-baseline --no-e2e --n-cubes 32 > gpurun_out/bench_el3.json 2> gpurun_out/bench_el3.log
BBWADG_LIB=paper_1808_08645_b200/native/em4/libbbwadg.so timeout 600 python bench.py --steps 1 --warmup 1 --no-sweep --no-config4 --no-cpu-baseline --no-e2e --n-cubes 8 --N 7 --M 2 --elastic 7:2:f64 > gpurun_out/bench_el3_em4.json 2> gpurun_out/bench_el3_em4.log
