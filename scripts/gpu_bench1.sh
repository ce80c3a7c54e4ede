set -x
python bench.py --n-cubes 20 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -3
python bench.py --steps 10 --warmup 3 --cpu-seconds 10 2>&1 | tail -3
