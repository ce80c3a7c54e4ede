#!/bin/bash
# 2D kernel after the register-resident LSRK state: parity suite + 2D bench lines; bench.py --halo peer under
# torchrun with 2 ranks sharing the one GPU (device-side stage barrier, gloo for the timing reductions)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 1200 python -m pytest tests/test_gpu_2d.py -q 2>&1 | tail -5 ) > gpurun_out/t2d_tests2.txt
timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep --no-config4 --elastic '' \
  --n-cubes 16 > gpurun_out/bench_2d2.json 2> gpurun_out/bench_2d2.log
timeout 900 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py \
  --gpus 2 --halo peer --n-cubes 24 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep --no-config4 \
  --elastic '' --two-d '' > gpurun_out/bench_peer2.json 2> gpurun_out/bench_peer2.log
echo "exit $?" >> gpurun_out/bench_peer2.log
