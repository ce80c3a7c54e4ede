# default bench line (config 5 + sweep + e2e + cpu baseline) and a full ncu capture of the N=M=9 stage kernel
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.log 2>&1; tail -1 gpurun_out/bench_full.log > gpurun_out/bench_full.json
ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 5 -c 1 -o gpurun_out/prof_n9 \
  python bench.py --config 3 --N 9 --M 9 --n-cubes 24 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-sweep > gpurun_out/ncu_n9.log 2>&1
tail -c 600 gpurun_out/bench_full.json
