#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 900 python -m pytest tests/test_gpu_graph.py -q 2>&1 | tail -8 ) > gpurun_out/graph_tests.txt
timeout 600 python scripts/graph_timing.py > gpurun_out/graph_timing.json 2>&1
( timeout 2700 python -m pytest tests -m gpu -q -x 2>&1 | tail -8 ) > gpurun_out/r2_tests_all4.txt
