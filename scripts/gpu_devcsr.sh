set -x
timeout 1200 python -m pytest tests -m gpu -q -x -k "device_offsets or loop_lists or first_call or dist" 2>&1 | tail -5
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-graph --no-sbp 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e'])"
