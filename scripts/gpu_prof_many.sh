# one --set full capture of each listed kernel (first instance after SKIP) + summary
TAG=${TAG:-pm}
K=${K:-k_apply_fix|k_win_mark|k_win_b|k_resolve|k_fuse_prep|k_all_points|k_apply_mark}
ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${SKIP:-30} -c ${CNT:-7} -o gpurun_out/pm_$TAG python bench.py --profile-only --steps 2 --warmup 3 > gpurun_out/pm_$TAG.log 2>&1; echo ncu $?
python scripts/prof_summary.py gpurun_out/pm_$TAG.ncu-rep 10 > gpurun_out/pm_$TAG.txt 2>&1
