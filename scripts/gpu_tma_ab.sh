#!/bin/bash
# sub-warp groups: cp.async (default) vs TMA bulk staging (tma8 variant) A/B at N = 3, 4 and racecheck of the
# default library at every sub-warp group shape
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in "3 1" "3 3" "4 2" "4 4"; do AB_NCUBE=56 timeout 600 python scripts/ab.py $c default tma8 2>&1 | tail -2; done > gpurun_out/ab_tma_subwarp.txt
L=gpurun_out/race_r2d.log
: > $L
for c in "3 1 2" "4 2 2" "2 2 2" "4 4 1"; do
  echo "== racecheck $c" >> $L
  timeout 900 compute-sanitizer --tool racecheck --num-cuda-barriers 128 --error-exitcode 9 python scripts/sanitize_case.py $c >> $L 2>&1
  echo "exit $?" >> $L
done
( timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "N=1 or N=2 or N=3 or N=4 or 1-1 or 2-2 or 3-1 or 4-2" 2>&1 | tail -3 ) > gpurun_out/subwarp_tests.txt
