#!/bin/bash
# compute-sanitizer on the elastic kernel (every group shape class) and the acoustic (2,2) rerun with
# enough barrier tracking slots for 32 sub-warp groups per CTA
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=gpurun_out/sanitizer_r2b.log
: > $L
for tool in racecheck synccheck memcheck; do
  for c in "3 1 2" "2 2 2" "7 2 2" "9 2 1" "5 3 2 f32" "4 0 2"; do
    echo "== elastic $tool $c" >> $L
    timeout 900 compute-sanitizer --tool $tool --num-cuda-barriers 128 --error-exitcode 9 python scripts/sanitize_elastic.py $c >> $L 2>&1
    echo "exit $?" >> $L
  done
  echo "== acoustic $tool 2 2 2 (--num-cuda-barriers 128)" >> $L
  timeout 900 compute-sanitizer --tool $tool --num-cuda-barriers 128 --error-exitcode 9 python scripts/sanitize_case.py 2 2 2 >> $L 2>&1
  echo "exit $?" >> $L
done
grep -E "^==|^exit|ERROR SUMMARY|RACECHECK SUMMARY|hazard|Warning" $L > gpurun_out/sanitizer_r2b_summary.txt
