set -x
LC_SOLE=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r2.py -m gpu -q -x -k "not C5" 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head -12
LC_SOLE=0 python bench.py --steps 10 --warmup 3 --no-sbp --no-cpu-baseline --no-e2e --no-graph 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('LC_SOLE=0', d['ms_per_step'], d['kernel_ms_per_step'])"
TAG=${TAG:-it} K="k_match_sole" CNT=1 SKIP=3 bash scripts/gpu_lines.sh
