# apply-pass change: parity (default + forced sole), dist, A/B timing, launch list
set -x
timeout 500 python -m pytest tests -m gpu -q -x -k "parity or r2 or dist" 2>&1 | tail -4
timeout 300 env LC_SOLE=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r2.py -m gpu -q -x -k "not C5" 2>&1 | tail -4
bash scripts/ab.sh; bash scripts/ab.sh
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_apply.csv python bench.py --profile-only --steps 2 --warmup 3 > /dev/null 2>&1; python scripts/launch_summary.py gpurun_out/launches_apply.csv | tail -16
