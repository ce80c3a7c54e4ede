# round-end evidence: default bench line, config-4 lines, ncu launch list and traffic/profile captures
# (the wavespeed study: python scripts/convergence.py --study wavespeed, ~10 min)
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_final.log 2>&1; tail -1 gpurun_out/bench_final.log > gpurun_out/bench_final.json
python bench.py --config 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep 2>&1 | tail -1 > gpurun_out/bench_c4_f64.json
python bench.py --config 4 --dtype f32 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep 2>&1 | tail -1 > gpurun_out/bench_c4_f32.json
bash scripts/gpu_launches.sh
bash scripts/gpu_traffic.sh
tail -c 400 gpurun_out/bench_final.json
