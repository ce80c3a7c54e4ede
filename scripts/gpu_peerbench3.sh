#!/bin/bash
# bench.py under torchrun with 2 ranks sharing the GPU: --halo auto (peer) end to end incl. e2e, and --halo nccl
# (expected to fail on one GPU: NCCL refuses two ranks on one device) to check the error path is clean
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29621 bench.py \
  --gpus 2 --n-cubes 24 --steps 3 --warmup 3 --no-cpu-baseline --no-sweep --no-config4 --elastic '' --two-d '' \
  > gpurun_out/bench_auto2.json 2> gpurun_out/bench_auto2.log
echo "exit $?" >> gpurun_out/bench_auto2.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sweep --no-config4 --elastic '' --two-d '' \
  > gpurun_out/bench_1gpu_c5.json 2> gpurun_out/bench_1gpu_c5.log
