TAG=${TAG:-ls}
ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --profile-only --steps 2 --warmup 3 > /dev/null 2>&1
python - <<'PY'
import csv, collections, re, os
tag=os.environ.get("TAG","ls")
rows=[r for r in csv.reader(open(f"gpurun_out/launches_{tag}.csv")) if len(r)>10]
h=rows[0]; ki=h.index("Kernel Name"); mi=h.index("Metric Name"); vi=h.index("Metric Value")
agg=collections.OrderedDict()
for r in rows[1:]:
    m=re.search(r"(k_\w+|at::\w+|\w+_kernel)", r[ki]); n=m.group(1) if m else r[ki][:30]
    agg.setdefault(n,collections.defaultdict(list))[r[mi]].append(float(r[vi].replace(",","")))
for n,d in agg.items():
    t=d.get("gpu__time_duration.sum",[0]); w=d.get("sm__warps_active.avg.pct_of_peak_sustained_active",[0]); g=d.get("launch__registers_per_thread",[0])
    print(f"{n:28s} n={len(t):3d} mean_us={sum(t)/len(t)/1000:8.2f} warps%={sum(w)/len(w):5.1f} regs={g[0]:.0f}")
PY
