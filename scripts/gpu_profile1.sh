# ncu launch list + one full capture of the stage kernel (config-5 shape, smaller mesh)
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_r1v2.csv \
  python bench.py --n-cubes 32 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 5 -c 1 -o gpurun_out/prof_stage_n7m4_r1v2 \
  python bench.py --n-cubes 32 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
