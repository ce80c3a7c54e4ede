#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python scripts/convergence_new_rows.py gpurun_out/convergence_new_rows.json > gpurun_out/convergence_new_rows.log 2>&1
