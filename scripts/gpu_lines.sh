# ncu --set full of k_project + k_match on one C5 step, then per-source-line warp-stall
# samples and executed instructions (scripts/ncu_lines.py) -> gpurun_out/lines_$TAG.txt
TAG=${TAG:-tmp}
K=${K:-k_project|k_match}
ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${SKIP:-6} -c ${CNT:-2} -o gpurun_out/lines_$TAG python bench.py --profile-only --steps 1 --warmup 3 > gpurun_out/lines_$TAG.log 2>&1; echo ncu $?
for k in $(echo "$K" | tr '|' ' '); do
  echo "=== $k" >> gpurun_out/lines_$TAG.txt
  python scripts/ncu_lines.py gpurun_out/lines_$TAG.ncu-rep "$k" 45 >> gpurun_out/lines_$TAG.txt 2>&1
done
tail -3 gpurun_out/lines_$TAG.txt
