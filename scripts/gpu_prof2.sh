# per-kernel device metrics (ncu) for each ab/*.so -> gpurun_out/p_<name>.csv
for f in ab/*.so; do
  n=$(basename $f .so)
  LC_LIB_PATH=$PWD/$f ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv --log-file gpurun_out/p_$n.csv -k regex:"k_project|k_match" -s 2 -c 2 python bench.py --profile-only --steps 1 --warmup 1 > /dev/null 2>&1
  echo "$n $?"
done
