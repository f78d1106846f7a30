set -x
timeout 1200 python -m pytest tests -m gpu -q -x -k "dist or point_range or first_call or parity_small or C5_full" 2>&1 | tail -4
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-graph --no-sbp --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['kernel_ms_per_step'])"
