# full GPU suite on the working tree's lib, then A/B timing of ab/*.so
set -x
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
bash scripts/ab.sh; bash scripts/ab.sh
