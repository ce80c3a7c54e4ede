#!/bin/bash
# A/B with the work queue on: LSRK state in registers (default) vs residual prefetched to L2 and re-read (r74, r53);
# queue vs static grid-stride at (5,3) and (9,9) (b53 / b99 = static, b53q / b99q = queue, same single-(N,M) builds)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/lsrk_ab.txt
AB_REPS=2 timeout 900 python scripts/ab.py 7 4 default r74 > $O 2>&1
AB_REPS=2 timeout 900 python scripts/ab.py 5 3 b53q r53 b53 >> $O 2>&1
AB_REPS=2 AB_NCUBE=44 timeout 600 python scripts/ab.py 9 9 b99q b99 >> $O 2>&1
cat $O
