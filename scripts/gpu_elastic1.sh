#!/bin/bash
# elastic kernel: first GPU parity run (+ smoke)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/el_smoke.txt 2>&1
( timeout 1500 python -m pytest tests/test_gpu_elastic.py -q -x 2>&1 | tail -30 ) > gpurun_out/el_tests.txt
