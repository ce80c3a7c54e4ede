#!/bin/bash
# round-2 re-entry baseline: GPU suite, smoke, the default bench line
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 ) > gpurun_out/r2_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.log
