# ncu --set full of the top kernel(s) for the current in-tree liblc.so
TAG=${TAG:-tmp}
K=${K:-k_project_match}
ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-3} -c ${CNT:-1} -o gpurun_out/prof_$TAG python bench.py --profile-only --steps 1 --warmup 3 > gpurun_out/prof_$TAG.log 2>&1; echo ncu $?
