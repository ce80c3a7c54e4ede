# ncu launch list (device time per stage-kernel launch) of the default bench configuration
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:stage_kernel -c 30 --csv \
  --log-file gpurun_out/launches_r1_final.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep \
  > gpurun_out/ncu_launches_final.log 2>&1
tail -3 gpurun_out/launches_r1_final.csv
