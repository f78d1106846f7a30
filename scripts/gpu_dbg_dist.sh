set -x
timeout 300 python -m pytest tests/test_gpu_dist.py -m gpu -q -x -k "S3" 2>&1 | grep -v "^$" | grep -i "assert\|passed\|failed\|Error" | head -12
LC_APPLY_SMEM=1 timeout 300 python -m pytest tests/test_gpu_dist.py -m gpu -q -x -k "S3" 2>&1 | tail -2
LC_STAMP_PREP=1 timeout 300 python -m pytest tests/test_gpu_dist.py -m gpu -q -x -k "S3" 2>&1 | tail -2
