#!/bin/bash
# fluxes after the volume elevation (BBW_FLUX_LATE=1) vs default; config-5 bench line of the default library
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
{ AB_NCUBE=56 timeout 600 python scripts/ab.py 7 4 default fl74 2>&1 | tail -2
  AB_NCUBE=56 timeout 600 python scripts/ab.py 5 3 default fl53 2>&1 | tail -2; } > gpurun_out/ab_fluxlate.txt
timeout 900 python bench.py --steps 5 --warmup 3 --no-sweep --no-config4 --no-cpu-baseline --elastic '' --two-d '' \
  > gpurun_out/bench_c5_fl.json 2> gpurun_out/bench_c5_fl.log
