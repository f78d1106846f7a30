#!/usr/bin/env python
"""Key metrics + top stall reasons + top source lines of every kernel in an ncu report:
  python scripts/prof_summary.py REP [N_LINES]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 12
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread", "launch__grid_size",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "lts__t_sector_hit_rate.pct"]
for r in rows[2:]:
    d = {h[i]: r[i] for i in range(len(h))}
    name = d["Kernel Name"]
    print("=" * 8, name[:90])
    print("  " + ", ".join(f"{k.split('__')[1] if '__' in k else k}={d.get(k)}" for k in KEYS))
    st = [(k, float(d[k])) for k in d if "smsp__pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")
          and d[k].replace(".", "", 1).isdigit()]
    tot = sum(x for _, x in st) or 1
    print("  stalls: " + ", ".join(f"{k.split('stalled_')[1]} {100 * x / tot:.0f}%" for k, x in sorted(st, key=lambda t: -t[1])[:6]))
    short = name.split("(")[0].split("::")[-1].split("<")[0]
    out = subprocess.run([sys.executable, "scripts/ncu_lines.py", rep, short, str(nl)], capture_output=True, text=True).stdout
    print("\n".join("  " + x for x in out.splitlines()[:nl + 1]))
