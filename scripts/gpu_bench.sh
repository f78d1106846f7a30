# full default bench line + reference arm (round-end style)
TAG=${TAG:-b}
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench $?; tail -3 gpurun_out/bench_$TAG.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>&1; echo ref $?; tail -1 gpurun_out/bench_ref_$TAG.json
