set -x
timeout 900 python -m pytest tests/test_gpu_pgo.py -m gpu -q -x 2>&1 | tail -3
GRAPHS="C3 C5" bash scripts/pgo_ab.sh 2>&1 | grep -v "cg cg_tol"
