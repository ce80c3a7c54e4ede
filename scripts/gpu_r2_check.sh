#!/bin/bash
# full GPU suite, racecheck of the acoustic (2,2) / (3,1) kernels after the TMA change, the default bench line
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -15 ) > gpurun_out/r2_tests_all2.txt
L=gpurun_out/race_r2c.log
: > $L
for c in "2 2 2" "1 1 2" "3 1 2"; do
  echo "== racecheck $c" >> $L
  timeout 900 compute-sanitizer --tool racecheck --num-cuda-barriers 128 --error-exitcode 9 python scripts/sanitize_case.py $c >> $L 2>&1
  echo "exit $?" >> $L
done
timeout 1500 python bench.py > gpurun_out/bench_full2.json 2> gpurun_out/bench_full2.log
