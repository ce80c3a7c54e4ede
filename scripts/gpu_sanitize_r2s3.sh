#!/bin/bash
# compute-sanitizer on the work-queue kernels: one CTA per SM (BBWADG_BLOCKS_PER_SM=1) so that units draw several
# tickets; sub-warp (3,1), whole-warp (7,4), 64-thread groups (9,9) acoustic; elastic (7,2) and (9,2)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=gpurun_out/sanitizer_r2s3.log
: > $L
export BBWADG_BLOCKS_PER_SM=1
for tool in racecheck synccheck memcheck; do
  for c in "3 1 6" "7 4 6" "9 9 4"; do
    echo "== acoustic $tool $c" >> $L
    timeout 900 compute-sanitizer --tool $tool --num-cuda-barriers 128 --error-exitcode 9 python scripts/sanitize_case.py $c >> $L 2>&1
    echo "exit $?" >> $L
  done
  for c in "7 2 4" "9 2 4"; do
    echo "== elastic $tool $c" >> $L
    timeout 900 compute-sanitizer --tool $tool --num-cuda-barriers 128 --error-exitcode 9 python scripts/sanitize_elastic.py $c >> $L 2>&1
    echo "exit $?" >> $L
  done
done
grep -E "^==|^exit|ERROR SUMMARY|RACECHECK SUMMARY|hazard|Warning|^ok" $L > gpurun_out/sanitizer_r2s3_summary.txt
cat gpurun_out/sanitizer_r2s3_summary.txt
