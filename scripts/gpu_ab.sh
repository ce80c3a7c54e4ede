# A/B the current library against named variants on config 5 (and optionally config 3 N=9)
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = default ]; then lib=$PWD/paper_1808_08645_b200/native/libbbwadg.so; else lib=$PWD/paper_1808_08645_b200/native/$v/libbbwadg.so; fi
  BBWADG_LIB=$lib python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v c5', '%.3e'%d['value'], 'frac', d['roofline']['frac'])"
  BBWADG_LIB=$lib python bench.py --config 3 --N 9 --M 9 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v c3N9', '%.3e'%d['value'], 'frac', d['roofline']['frac'])"
done; done
