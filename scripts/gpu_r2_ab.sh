#!/bin/bash
# round-2 A/B: parity suite on the default library, then default vs variants at several (N, M)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
VARS=${VARS:-v4}
CASES=${CASES:-"7 4;5 3;9 9;3 1"}
( timeout 900 python -m pytest tests -m gpu -x -q -k "${TESTK:-wadg_apply or rhs_parity or steps_parity}" 2>&1 | tail -5 ) > gpurun_out/r2_tests.txt
IFS=';' read -ra CS <<< "$CASES"
for c in "${CS[@]}"; do
  AB_NCUBE=${AB_NCUBE:-56} timeout 600 python scripts/ab.py $c default $VARS 2>&1 | tail -4
done > gpurun_out/r2_ab.txt
