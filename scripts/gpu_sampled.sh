#!/bin/bash
# full-size sampled parity of the elastic and 2D bench workloads, then the whole GPU suite
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 1500 python -m pytest tests/test_gpu_elastic.py tests/test_gpu_2d.py -q -k "full_size" 2>&1 | tail -15 ) > gpurun_out/sampled_tests.txt
( timeout 2700 python -m pytest tests -m gpu -q 2>&1 | tail -8 ) > gpurun_out/r2_tests_all3.txt
