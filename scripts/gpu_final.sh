# round-end evidence: default bench line, ncu traffic/profile captures, wavespeed-frequency study
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_final.log 2>&1; tail -1 gpurun_out/bench_final.log > gpurun_out/bench_final.json
python bench.py --config 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep 2>&1 | tail -1 > gpurun_out/bench_c4_f64.json
python bench.py --config 4 --dtype f32 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep 2>&1 | tail -1 > gpurun_out/bench_c4_f32.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_final.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep > gpurun_out/ncu_launches.log 2>&1
bash scripts/gpu_traffic.sh
python scripts/convergence.py --study wavespeed > gpurun_out/wavespeed.log 2>&1; cp profiles/wavespeed_r1.json gpurun_out/ 2>/dev/null
tail -c 400 gpurun_out/bench_final.json
