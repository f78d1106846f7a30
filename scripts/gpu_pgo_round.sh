# full GPU tests, bench line, launch list and ncu of the PGO kernel (C3 graph)
set -x
TAG=${TAG:-r01}
python -m pytest tests -m gpu -q -x 2>&1 | tail -5
LC_LIB_PATH=$PWD/ab/pgotim.so timeout 300 python scripts/pgo_timing.py C2 C3 C5
python bench.py --steps 10 --warmup 3 --cpu-seconds 15 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --profile-only --steps 2 --warmup 3 > /dev/null 2>&1; echo ncu1 $?
ncu --set full --clock-control none --import-source on -k regex:k_pgo -c 1 -o gpurun_out/pgo_$TAG python scripts/pgo_probe.py C3 > gpurun_out/ncu_pgo_$TAG.log 2>&1; echo ncu2 $?
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>&1; tail -1 gpurun_out/bench_ref_$TAG.json
