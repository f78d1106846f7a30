#!/usr/bin/env python
"""Per-kernel table of a `--set full` capture of every liblc kernel of one step:
  python scripts/ncu_step_summary.py REP OUT.md TITLE"""
import csv
import io
import subprocess
import sys

rep, out_md, title = sys.argv[1], sys.argv[2], sys.argv[3]
mets = ("gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,"
        "launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,"
        "smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct")
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", mets],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u = rows[0], rows[1]


def mb(d, k):
    v = float(d[k].replace(",", ""))
    return v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u[h.index(k)], 1e-6)


md = [f"# {title}", "", "ncu `--set full --clock-control none`; each kernel replayed alone from a cold L2,",
      "so the times are per launch and serialised (the bench's CUDA-event times are authoritative).", "",
      "| kernel | us | DRAM read MB | DRAM write MB | GB/s | grid | regs | warps active % | issue active % | L2 hit % |",
      "|---|---|---|---|---|---|---|---|---|---|"]
for r in rows[2:]:
    d = dict(zip(h, r))
    name = d["Kernel Name"].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
    us = float(d["gpu__time_duration.sum"].replace(",", ""))
    rd, wr = mb(d, "dram__bytes_read.sum"), mb(d, "dram__bytes_write.sum")
    md.append(f"| {name} | {us:.1f} | {rd:.1f} | {wr:.1f} | {(rd + wr) * 1e-3 / (us * 1e-6):.0f} | "
              f"{d['launch__grid_size']} | {d['launch__registers_per_thread']} | "
              f"{float(d['sm__warps_active.avg.pct_of_peak_sustained_active']):.1f} | "
              f"{float(d['smsp__issue_active.avg.pct_of_peak_sustained_active']):.1f} | "
              f"{float(d['lts__t_sector_hit_rate.pct']):.1f} |")
open(out_md, "w").write("\n".join(md) + "\n")
print("\n".join(md))
