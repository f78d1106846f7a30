# A/B timing of alternative liblc builds under ab/*.so (bench kernel_ms_per_step)
for f in ab/*.so; do
  echo "== $f"
  LC_LIB_PATH=$PWD/$f python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-sbp 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['kernel_ms_per_step'])"
done
