#!/usr/bin/env python
"""Per-kernel mean duration (us) from an ncu --metrics gpu__time_duration.sum --csv launch list:
  python scripts/launch_summary.py launches.csv"""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.OrderedDict()
for r in rows[1:]:
    m = re.search(r"(k_\w+|at::\w+|\w+_kernel)", r[ki])
    n = m.group(1) if m else r[ki][:40]
    v = float(r[vi].replace(",", ""))
    v = v / 1000.0 if r[ui] in ("ns", "nsecond") else (v * 1000.0 if r[ui] in ("ms", "msecond") else v)
    agg.setdefault(n, []).append(v)
for n, v in agg.items():
    print(f"{n:28s} n={len(v):4d} mean_us={sum(v) / len(v):9.2f} total_us={sum(v):10.1f}")
