# parity tests + config-5 and config-3 (N=9,M=9) bench lines for the in-tree library
set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c5 N7M4', '%.3e'%d['value'], 'frac', d['roofline']['frac'], 'ms/step', round(d['ms_per_step'],2), d['clocks'])"
python bench.py --config 3 --N 9 --M 9 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c3 N9M9', '%.3e'%d['value'], 'frac', d['roofline']['frac'])"
python bench.py --config 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c4 N5M3', '%.3e'%d['value'], 'frac', d['roofline']['frac'])"
