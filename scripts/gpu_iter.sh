# iteration: parity (default + forced sole mode), short bench, launch list
set -x
TAG=${TAG:-it}
timeout 400 python -m pytest tests -m gpu -q -x -k "parity or r2" 2>&1 | tail -4
timeout 300 env LC_SOLE=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r2.py -m gpu -q -x -k "not C5" 2>&1 | tail -4
python bench.py --steps 10 --warmup 3 --no-sbp --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err
python -c "import json; d=json.load(open('gpurun_out/bench_$TAG.json')); print(d['ms_per_step'], d['kernel_ms_per_step'], d['graph'], d['roofline']['frac'])"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --profile-only --steps 2 --warmup 3 > /dev/null 2>&1; python scripts/launch_summary.py gpurun_out/launches_$TAG.csv | tail -14
