#!/bin/bash
# full ncu capture of the config-5-shaped stage kernel for several library variants
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = default ]; then lib=$PWD/paper_1808_08645_b200/native/libbbwadg.so; else lib=$PWD/paper_1808_08645_b200/native/$v/libbbwadg.so; fi
  BBWADG_LIB=$lib timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 5 -c 1 \
    -o gpurun_out/prof_$v python bench.py --n-cubes 32 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep \
    > gpurun_out/ncu_$v.log 2>&1
done
