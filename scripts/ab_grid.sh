for g in 64x48 96x72 128x96 160x120; do
  echo "== grid $g"
  LC_GRID=$g python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['kernel_ms_per_step'], d['config']['candidates_per_step'])"
done
