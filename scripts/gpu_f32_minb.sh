#!/bin/bash
# fp32 occupancy: the fp32 element block is half the fp64 one, so shared memory allows 8+ CTAs per SM; the
# launch bounds (MINB) cap registers instead.  A/B of MINB 6 / 8 against the default at (5,3) and (7,4) fp32
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
{ AB_DTYPE=f32 AB_NCUBE=56 timeout 600 python scripts/ab.py 5 3 default m6_53 m8_53 2>&1 | tail -3
  AB_DTYPE=f32 AB_NCUBE=56 timeout 600 python scripts/ab.py 7 4 default m6_74 m8_74 2>&1 | tail -3; } > gpurun_out/ab_f32_minb.txt
