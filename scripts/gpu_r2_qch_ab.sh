#!/bin/bash
# work-queue chunk A/B (QCH unit-batches per ticket): config-5 bench (default QCH=2, c1_74, c4_74, b74 static),
# ab.py at (5,3) n=64 and (9,9) n=44 (b53/b99 static, b53q/b99q QCH=1, default QCH=2, c4_* QCH=4)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
lib() { if [ $1 = default ]; then echo paper_1808_08645_b200/native/libbbwadg.so; else echo paper_1808_08645_b200/native/$1/libbbwadg.so; fi; }
for rep in 1 2; do
for v in default c1_74 c4_74 b74; do
  BBWADG_LIB=$(lib $v) timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep --no-config4 \
    --elastic '' --two-d '' > gpurun_out/qch_bench_${v}_$rep.json 2> /dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/qch_bench_${v}_$rep.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
done
O=gpurun_out/qch_ab.txt
AB_REPS=2 timeout 900 python scripts/ab.py 5 3 b53 b53q default c4_53 > $O 2>&1
AB_REPS=2 AB_NCUBE=44 timeout 900 python scripts/ab.py 9 9 b99 b99q default c4_99 >> $O 2>&1
cat $O
