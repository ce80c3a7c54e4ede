#!/bin/bash
# N = 8: 5 CTAs per SM (launch bounds MINB=5, 96 registers) vs 4 (128 registers), config-3 mesh n=44
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
AB_REPS=2 AB_NCUBE=44 timeout 900 python scripts/ab.py 8 8 m4_88 m5_88 > gpurun_out/minb8_ab.txt 2>&1
AB_REPS=2 AB_NCUBE=44 timeout 900 python scripts/ab.py 8 2 m4_82 m5_82 >> gpurun_out/minb8_ab.txt 2>&1
cat gpurun_out/minb8_ab.txt
