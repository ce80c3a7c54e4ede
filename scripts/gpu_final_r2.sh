#!/bin/bash
# round-2 final evidence: ncu launch list of the default (config-5) bench, one --set full capture of the
# config-5 stage kernel (DRAM traffic for roofline.traffic), DRAM per launch at configs 4 / 3, and --set full
# captures of the elastic (7,2) and 2D (7,4) kernels
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ONLY5="--no-e2e --no-cpu-baseline --no-sweep --no-config4 --elastic '' --two-d ''"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:stage_kernel -c 30 --csv \
  --log-file gpurun_out/r2_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep \
  --no-config4 --elastic '' --two-d '' > gpurun_out/ncu_launches_r2.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 5 -c 1 -o gpurun_out/prof_r2_c5 \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-sweep --no-config4 --elastic '' --two-d '' \
  > gpurun_out/ncu_r2_c5.log 2>&1
ncu -i gpurun_out/prof_r2_c5.ncu-rep --page raw --csv > gpurun_out/traffic_N7M4f64.csv 2>/dev/null
python scripts/ncu_phases.py gpurun_out/prof_r2_c5.ncu-rep paper_1808_08645_b200/native/libbbwadg.so "StageCfgILi7ELi4Ed" 4088832 \
  > gpurun_out/phases_r2_c5.txt 2>&1
for cfg in "4 5 3 f64" "4 5 3 f32" "3 9 9 f64"; do
  set -- $cfg
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:stage_kernel -s 5 -c 1 --csv --log-file gpurun_out/traffic_N$2M$3$4.csv \
    python bench.py --config $1 --N $2 --M $3 --dtype $4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-sweep \
    --no-config4 --elastic '' --two-d '' > gpurun_out/ncu_traffic_N$2M$3$4.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:elastic_stage -s 3 -c 1 -o gpurun_out/prof_r2_el72 \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-sweep --no-config4 --n-cubes 8 --elastic 7:2:f64 \
  --two-d '' > gpurun_out/ncu_r2_el72.log 2>&1
ncu -i gpurun_out/prof_r2_el72.ncu-rep --page raw --csv > gpurun_out/el72_raw_final.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage2d -s 3 -c 1 -o gpurun_out/prof_r2_2d74 \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-sweep --no-config4 --n-cubes 8 --elastic '' \
  --two-d 7:4:f64 > gpurun_out/ncu_r2_2d74.log 2>&1
ncu -i gpurun_out/prof_r2_2d74.ncu-rep --page raw --csv > gpurun_out/t2d74_raw.csv 2>/dev/null
mkdir -p /tmp/ncu_reps && mv gpurun_out/*.ncu-rep /tmp/ncu_reps/ 2>/dev/null  # keep gpurun_out under 64 MiB
ls -la gpurun_out | tail -20
