# ncu --set full of the non-matching kernels of the C5 step + bench e2e distribution
set -x
ncu --set full --clock-control none --import-source on -k regex:"k_apply_fix|k_apply_mark|k_win_mark|k_win_b|k_fuse_prep|k_all_points" -s 12 -c 6 -o gpurun_out/rest_r02 python bench.py --profile-only --steps 1 --warmup 3 > gpurun_out/rest_r02.log 2>&1; echo ncu $?
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-graph --no-sbp > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; echo bench $?
python -c "import json; d=json.load(open('gpurun_out/bench_e2e.json')); print(d['ms_per_step'], d['e2e'])"
