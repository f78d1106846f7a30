set -x
timeout 600 python -m pytest tests/test_gpu_pgo.py -m gpu -q -x -k "cyclic and C5" 2>&1 | grep -E "Error|assert|Mismatch|Max|x:|y:|^E" | head -30
ncu --set full --clock-control none --import-source on -k regex:k_pgo -c 1 -o gpurun_out/pgo_cr python scripts/pgo_one.py C2 cr 3 > gpurun_out/pgo_cr.log 2>&1; echo ncu $?
python scripts/ncu_lines.py gpurun_out/pgo_cr.ncu-rep k_pgo 60 > gpurun_out/pgo_cr.txt 2>&1
head -70 gpurun_out/pgo_cr.txt
