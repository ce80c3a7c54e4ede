#!/bin/bash
# full GPU suite + compute-sanitizer + M=0 fast-path A/B + M<N convergence study
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -15 ) > gpurun_out/r2_tests_full.txt
./scripts/gpu_sanitize.sh
for c in "7 0" "5 0" "3 0" "7 1"; do AB_NCUBE=56 timeout 600 python scripts/ab.py $c default m0slow 2>&1 | tail -2; done > gpurun_out/r2_ab_m0.txt
timeout 1200 python scripts/convergence.py --study mlessn --n 4 8 16 --out gpurun_out/convergence_mlessn_r2.json > gpurun_out/conv_mlessn.log 2>&1
