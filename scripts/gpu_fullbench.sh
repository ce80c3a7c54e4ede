#!/bin/bash
# the default bench line (what the driver runs), timed end to end
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
s=$(date +%s)
timeout 1800 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.log
echo "bench wall seconds: $(( $(date +%s) - s ))" >> gpurun_out/bench_full.log
