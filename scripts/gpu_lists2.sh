set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "loop_lists or device_offsets or pipelined" 2>&1 | tail -2
python scripts/lists_dev_probe.py
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-graph --no-sbp 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['kernel_ms_per_step'])"
