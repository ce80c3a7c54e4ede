#!/bin/bash
# peer-read halo: new tests first, then the whole GPU suite, then a quick config-5 bench (no regression)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "peer" 2>&1 | tail -30 ) > gpurun_out/peer_tests.txt
( timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -15 ) > gpurun_out/r2_tests_all.txt
timeout 900 python bench.py --steps 5 --warmup 3 --no-sweep --no-config4 --no-cpu-baseline --elastic '' > gpurun_out/bench_peer.json 2> gpurun_out/bench_peer.log
