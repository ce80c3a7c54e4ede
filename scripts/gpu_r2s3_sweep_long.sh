#!/bin/bash
# SURVEY 8(d) config-3 protocol for the order sweep: 10 warm-up + 100 timed LSRK steps per N (M = N, n = 44,
# 511,104 tets, Gaussian pulse), plus the fixed-M=1 rows; then the whole -m gpu suite and smoke on this library
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-config4 --elastic '' --two-d '' \
  --sweep-warmup 10 --sweep-steps 100 > gpurun_out/sweep_long.json 2> gpurun_out/sweep_long.err
echo "sweep exit $?" >> gpurun_out/sweep_long.err
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/final2_gpu_suite.txt 2>&1
echo "pytest exit $?" >> gpurun_out/final2_gpu_suite.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2_smoke.txt 2>&1
echo "smoke exit $?" >> gpurun_out/final2_smoke.txt
tail -2 gpurun_out/final2_gpu_suite.txt; tail -1 gpurun_out/final2_smoke.txt; tail -1 gpurun_out/sweep_long.err
