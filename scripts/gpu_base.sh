# round-start baseline on the GPU box: tests, bench line, launch list
set -x
TAG=${TAG:-r02a}
python -m pytest tests -m gpu -q -x 2>&1 | tail -6
python bench.py --steps 10 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --profile-only --steps 2 --warmup 3 > /dev/null 2>&1; echo ncu1 $?
