#!/bin/bash
# the final default bench line of round 2 (what the driver runs), plus smoke
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.txt 2>&1
s=$(date +%s)
timeout 1800 python bench.py > gpurun_out/bench_r2_final.json 2> gpurun_out/bench_r2_final.log
echo "bench wall seconds: $(( $(date +%s) - s ))" >> gpurun_out/bench_r2_final.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_final.json 2> gpurun_out/bench_ref_final.log
