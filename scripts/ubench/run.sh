#!/bin/bash
# microbenchmarks of SM resources + a baseline config-5 bench line (round-2 start)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/ub_smi.txt
./scripts/ubench/ubench > gpurun_out/ubench.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/bench_r2_base.json 2> gpurun_out/bench_r2_base.log
