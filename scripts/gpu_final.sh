# end-of-round evidence: full GPU tests + smoke, bench line, reference arm, launch list,
# ncu of the matching stage and of the PGO kernel
set -x
TAG=${TAG:-r01}
python -m pytest tests -m gpu -q 2>&1 | tail -4
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 10 --warmup 3 --cpu-seconds 15 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>&1; tail -1 gpurun_out/bench_ref_$TAG.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --profile-only --steps 2 --warmup 3 > /dev/null 2>&1; echo ncu1 $?
ncu --set full --clock-control none --import-source on -k regex:'k_project|k_match' -s 6 -c 2 -o gpurun_out/match_$TAG python bench.py --profile-only --steps 1 --warmup 3 > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu2 $?
ncu --set full --clock-control none --import-source on -k regex:k_pgo -c 1 -o gpurun_out/pgo_$TAG python scripts/pgo_probe.py C3 > gpurun_out/ncu_pgo_$TAG.log 2>&1; echo ncu3 $?
