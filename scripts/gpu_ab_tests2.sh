# parity (fuse paths) on the working tree's lib, then A/B timing old vs new
set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "parity or edges or r2 or dist or graph" 2>&1 | tail -4
bash scripts/ab.sh; bash scripts/ab.sh
