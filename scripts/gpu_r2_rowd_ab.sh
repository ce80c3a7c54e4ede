#!/bin/bash
# A/B of the round-2 session-3 changes: dynamic work queue (BBW_DYNQ) and row-owned lift layers (BBW_ROWD)
# default = both on; b<NM> = both off (the previous kernel); q74 = queue only.  Parity first.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/rowd_ab.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/rowd_parity.txt 2>&1
echo "parity exit $?" >> gpurun_out/rowd_parity.txt
tail -2 gpurun_out/rowd_parity.txt
AB_REPS=2 timeout 900 python scripts/ab.py 7 4 b74 default q74 > $O 2>&1
AB_REPS=2 timeout 600 python scripts/ab.py 5 3 b53 default >> $O 2>&1
AB_REPS=2 AB_NCUBE=44 timeout 600 python scripts/ab.py 9 9 b99 default >> $O 2>&1
cat $O
ONLY5="--no-e2e --no-cpu-baseline --no-sweep --no-config4 --elastic '' --two-d ''"
for v in default b74 q74; do
  if [ $v = default ]; then lib=paper_1808_08645_b200/native/libbbwadg.so; else lib=paper_1808_08645_b200/native/$v/libbbwadg.so; fi
  BBWADG_LIB=$lib timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:stage_kernel -s 5 -c 1 --csv --log-file gpurun_out/rowd_dram_$v.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-sweep --no-config4 --elastic '' --two-d '' \
    > gpurun_out/rowd_dram_$v.log 2>&1
  grep -E "dram__bytes|duration|wavefronts|hit_rate" gpurun_out/rowd_dram_$v.csv | awk -F'","' '{print "'$v'", $(NF-2), $NF}'
done
