#!/bin/bash
# round-2 session-3 evidence with the work queue: ncu captures (scripts/gpu_final_r2.sh), traffic.json refreshed
# on the box so the bench line's roofline.traffic is this kernel's, full -m gpu suite, smoke, default bench line
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash scripts/gpu_final_r2.sh > gpurun_out/final_ncu_driver.log 2>&1
python scripts/make_traffic_json.py gpurun_out > gpurun_out/traffic_json.log 2>&1
cp profiles/traffic.json gpurun_out/traffic_new.json
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/final_gpu_suite.txt 2>&1
echo "pytest exit $?" >> gpurun_out/final_gpu_suite.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.txt 2>&1
echo "smoke exit $?" >> gpurun_out/final_smoke.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/final_smi.txt
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
echo "bench exit $?" >> gpurun_out/final_bench.err
tail -2 gpurun_out/final_gpu_suite.txt; tail -1 gpurun_out/final_smoke.txt
