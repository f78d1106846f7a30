set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -5
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -2
