# ncu --set full of one lc_pgo_sim3 launch (C2 graph), source-level stall sampling
TAG=${TAG:-pgo}
ncu --set full --clock-control none --import-source on -k regex:k_pgo -c 1 -o gpurun_out/pgo_$TAG python scripts/pgo_probe.py ${GRAPH:-C2} > gpurun_out/ncu_pgo_$TAG.log 2>&1; echo ncu $?; tail -3 gpurun_out/ncu_pgo_$TAG.log
