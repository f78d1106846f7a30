# ncu --set full of every liblc kernel of one bench step (the 4th: after 3 warm-ups)
TAG=${TAG:-all}
set -x
ncu --set full --clock-control none --import-source on -k regex:'^k_(win|all|fuse|apply|project|match)' -s 33 -c 11 -o gpurun_out/step_$TAG python bench.py --profile-only --steps 1 --warmup 3 > gpurun_out/ncu_step_$TAG.log 2>&1; echo ncu $?; tail -3 gpurun_out/ncu_step_$TAG.log
