#!/bin/bash
# full GPU suite on the default library + A/B against variants (config-5 (N, M) and others)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -15 ) > gpurun_out/r2_tests.txt
IFS=';' read -ra CS <<< "${CASES:-7 4}"
for c in "${CS[@]}"; do
  AB_NCUBE=${AB_NCUBE:-56} timeout 600 python scripts/ab.py $c default ${VARS:-v4} 2>&1 | tail -4
done > gpurun_out/r2_ab.txt
