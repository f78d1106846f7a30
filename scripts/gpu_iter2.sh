set -x
TAG=${TAG:-it}
python -m pytest tests -m gpu -q -x -k "parity or r2" 2>&1 | tail -3
LC_SOLE=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r2.py -m gpu -q -x -k "not C5" 2>&1 | tail -3
bash scripts/ab.sh
TAG=$TAG K="k_project|k_match_sole" bash scripts/gpu_lines.sh
