set -x
timeout 400 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 180 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1
