# A/B incl. e2e: ms_per_step, e2e ms, kernel families of each ab/*.so
for f in ab/*.so; do
  echo "== $f"
  LC_LIB_PATH=$PWD/$f python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-graph --no-sbp 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], 'e2e', d['e2e']['ms_per_step'], d['kernel_ms_per_step'])"
done
