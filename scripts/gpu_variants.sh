# compare tuning variants of libbbwadg.so on the config-5 bench (no e2e / cpu baseline)
python __graft_entry__.py smoke 2>&1 | tail -1
for v in default tg64 t256 tg64et2 et2; do
  if [ "$v" = default ]; then lib=paper_1808_08645_b200/native/libbbwadg.so; else lib=paper_1808_08645_b200/native/$v/libbbwadg.so; fi
  BBWADG_LIB=$PWD/$lib python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.3e'%d['value'], 'frac', d['roofline']['frac'], 'ms/step', round(d['ms_per_step'],1))"
done
