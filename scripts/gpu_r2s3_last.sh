#!/bin/bash
# last validation of the round: whole -m gpu suite, smoke, default bench line
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/last_gpu_suite.txt 2>&1
echo "pytest exit $?" >> gpurun_out/last_gpu_suite.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last_smoke.txt 2>&1
echo "smoke exit $?" >> gpurun_out/last_smoke.txt
timeout 900 python bench.py > gpurun_out/last_bench.json 2> gpurun_out/last_bench.err
echo "bench exit $?" >> gpurun_out/last_bench.err
tail -2 gpurun_out/last_gpu_suite.txt; tail -1 gpurun_out/last_smoke.txt; tail -1 gpurun_out/last_bench.err
