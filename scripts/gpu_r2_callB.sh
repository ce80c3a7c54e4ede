#!/bin/bash
# round-2 evidence: sanitizer reruns at 32 groups/CTA, TMEM alloc concurrency probe, product re-anneal A/B,
# the default bench line, its ncu launch list, DRAM traffic per stage launch (config 5/4/3)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in racecheck synccheck; do
  echo "== $tool 2 2 2 --num-cuda-barriers 128" >> gpurun_out/sanitizer_r2b.log
  timeout 900 compute-sanitizer --tool $tool --num-cuda-barriers 128 --error-exitcode 9 python scripts/sanitize_case.py 2 2 2 >> gpurun_out/sanitizer_r2b.log 2>&1
  echo "exit $?" >> gpurun_out/sanitizer_r2b.log
done
./scripts/ubench/tmem_alloc > gpurun_out/tmem_alloc.txt 2>&1
for c in "7 4" "5 3"; do AB_NCUBE=56 timeout 600 python scripts/ab.py $c default oldanneal 2>&1 | tail -2; done > gpurun_out/r2_ab_anneal.txt
timeout 900 python bench.py > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/r2_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep --no-config4 > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 5 -c 1 -o gpurun_out/prof_r2_c5 \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-sweep --no-config4 > gpurun_out/ncu_r2_c5.log 2>&1
ncu -i gpurun_out/prof_r2_c5.ncu-rep --page raw --csv > gpurun_out/traffic_N7M4f64.csv 2>/dev/null
for cfg in "4 5 3 f64" "4 5 3 f32" "3 9 9 f64"; do
  set -- $cfg
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:stage_kernel -s 5 -c 1 --csv --log-file gpurun_out/traffic_N$2M$3$4.csv \
    python bench.py --config $1 --N $2 --M $3 --dtype $4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-sweep --no-config4 \
    > gpurun_out/ncu_traffic_N$2M$3$4.log 2>&1
done
