#!/bin/bash
# dynamic work queue (BBW_DYNQ): full GPU suite, then config-5 bench A/B (default = queue, b74 = static grid-stride,
# q74 = queue without the ticket prefetch), elastic (7,2) A/B (b72 = static), ncu DRAM bytes of each
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/dynq_gpu_suite.txt 2>&1
echo "pytest exit $?" >> gpurun_out/dynq_gpu_suite.txt
tail -2 gpurun_out/dynq_gpu_suite.txt
ONLY5="--no-e2e --no-cpu-baseline --no-sweep --no-config4 --elastic '' --two-d ''"
lib() { if [ $1 = default ]; then echo paper_1808_08645_b200/native/libbbwadg.so; else echo paper_1808_08645_b200/native/$1/libbbwadg.so; fi; }
for rep in 1 2; do
for v in default b74 q74; do
  BBWADG_LIB=$(lib $v) timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep --no-config4 \
    --elastic '' --two-d '' > gpurun_out/dynq_bench_${v}_$rep.json 2> /dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/dynq_bench_${v}_$rep.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'])"
done
done
for v in default b72; do
  BBWADG_LIB=$(lib $v) timeout 600 python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-sweep --no-config4 \
    --elastic 7:2:f64 --two-d '' > gpurun_out/dynq_el_${v}.json 2> /dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/dynq_el_${v}.json').read().strip().splitlines()[-1]); print('$v elastic', d['elastic'])" | cut -c1-400
  BBWADG_LIB=$(lib $v) timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:elastic_stage -s 3 -c 1 --csv --log-file gpurun_out/dynq_el_dram_$v.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-sweep --no-config4 --n-cubes 8 --elastic 7:2:f64 --two-d '' \
    > /dev/null 2>&1
  grep -E "dram__bytes|duration" gpurun_out/dynq_el_dram_$v.csv | awk -F'","' '{print "'$v'", $(NF-2), $NF}'
done
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:stage_kernel -s 5 -c 1 --csv --log-file gpurun_out/dynq_dram_default.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-sweep --no-config4 --elastic '' --two-d '' > /dev/null 2>&1
grep -E "dram__bytes|duration|wavefronts|hit_rate" gpurun_out/dynq_dram_default.csv | awk -F'","' '{print "default", $(NF-2), $NF}'
