# DRAM bytes of one config-5 stage launch for library variants (ncu), plus their A/B speed
mkdir -p gpurun_out
for v in "$@"; do
  BBWADG_LIB=$PWD/paper_1808_08645_b200/native/$v/libbbwadg.so ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:stage_kernel -s 5 -c 1 --csv --log-file gpurun_out/dram_$v.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-sweep > /dev/null 2>&1
  echo "== $v"; grep -o '"dram__bytes_[a-z]*.sum","[A-Za-z]*","[0-9.,]*"\|"gpu__time_duration.sum","[a-z]*","[0-9.,]*"\|"lts__t_sector_hit_rate.pct","%","[0-9.,]*"' gpurun_out/dram_$v.csv
done
AB_REPS=1 python scripts/ab.py 7 4 "$@"
