# e2e probe + ncu --set full of k_project and k_match (r02 profiles)
set -x
timeout 300 python scripts/e2e_probe.py 2>&1 | tail -12
timeout 300 python scripts/lists_time.py 2>&1 | tail -8
ncu --set full --clock-control none --import-source on -k regex:"k_project|k_match" -s 2 -c 2 -o gpurun_out/full_r02 python bench.py --profile-only --steps 1 --warmup 3 > gpurun_out/full_r02.log 2>&1; echo ncu $?
