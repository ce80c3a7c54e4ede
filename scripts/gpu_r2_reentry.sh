#!/bin/bash
# re-entry check after a container rebuild: full -m gpu suite + default bench line
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/reentry_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/reentry_gpu_suite.txt 2>&1
echo "pytest exit $?" >> gpurun_out/reentry_gpu_suite.txt
timeout 900 python bench.py > gpurun_out/reentry_bench.json 2> gpurun_out/reentry_bench.err
echo "bench exit $?" >> gpurun_out/reentry_bench.err
tail -3 gpurun_out/reentry_gpu_suite.txt
