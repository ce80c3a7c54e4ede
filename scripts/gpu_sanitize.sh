#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck on small runs of every kernel shape class:
# (3,1) sub-warp groups (BASELINE config 1), (2,2) 4-lane groups, (7,4) whole warp, (9,9) two-warp groups
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in racecheck synccheck memcheck; do
  for c in "3 1 2" "2 2 2" "7 4 2" "9 9 1" "5 3 2 f32"; do
    echo "== $tool $c" >> gpurun_out/sanitizer_r2.log
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_case.py $c \
      >> gpurun_out/sanitizer_r2.log 2>&1
    echo "exit $?" >> gpurun_out/sanitizer_r2.log
  done
done
grep -E "^==|^exit|ERROR SUMMARY|RACECHECK SUMMARY|hazard" gpurun_out/sanitizer_r2.log | tail -60 > gpurun_out/sanitizer_r2_summary.txt
