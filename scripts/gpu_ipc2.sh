#!/bin/bash
# peer-read halo across processes with the device-side epoch barrier (bbwadg_run alone) and with host barriers
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "ipc or peer" 2>&1 | tail -30 ) > gpurun_out/ipc2_tests.txt
