#!/bin/bash
# 2D kernel: first GPU parity run; racecheck of the acoustic (2,2) kernel with 16 instead of 32 sub-warp groups
# per CTA (BBW_T=64 variant: same TG = 4 code, half the mbarriers) to separate the tool's tracking limit from
# a real hazard
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 1500 python -m pytest tests/test_gpu_2d.py -q -x 2>&1 | tail -30 ) > gpurun_out/t2d_tests.txt
BBWADG_LIB=paper_1808_08645_b200/native/t64/libbbwadg.so timeout 900 compute-sanitizer --tool racecheck \
  --num-cuda-barriers 128 --error-exitcode 9 python scripts/sanitize_case.py 2 2 2 > gpurun_out/race_t64.log 2>&1
echo "exit $?" >> gpurun_out/race_t64.log
