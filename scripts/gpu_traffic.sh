# DRAM traffic per stage-kernel launch at the bench configurations (ncu, one launch each),
# plus one `--set full` capture of the config-5 stage kernel.  Writes gpurun_out/traffic_*.csv.
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 5 -c 1 -o gpurun_out/prof_c5_full \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-sweep > gpurun_out/ncu_c5_full.log 2>&1
ncu -i gpurun_out/prof_c5_full.ncu-rep --page raw --csv > gpurun_out/traffic_N7M4f64.csv 2>/dev/null
for cfg in "4 5 3 f64" "4 5 3 f32" "3 9 9 f64"; do
  set -- $cfg
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:stage_kernel -s 5 -c 1 --csv --log-file gpurun_out/traffic_N$2M$3$4.csv \
    python bench.py --config $1 --N $2 --M $3 --dtype $4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-sweep \
    > gpurun_out/ncu_traffic_N$2M$3$4.log 2>&1
done
ls -la gpurun_out | tail
