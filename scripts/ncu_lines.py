#!/usr/bin/env python
"""Per-source-line warp-stall samples / instructions of one kernel in an ncu report:
  python scripts/ncu_lines.py REP KERNEL_REGEX [N]"""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 35
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kre,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[2]
iS, iI = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


lines, fname = [], ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) < len(h) or r[0] in ("", "Line No"):
        continue
    lines.append([f"{fname}:{r[0]}", r[1][:100], num(r[iS]), num(r[iI])])
tot = sum(x[2] for x in lines) or 1
toti = sum(x[3] for x in lines) or 1
print("total samples", tot, "warp instructions", toti)
for x in sorted(lines, key=lambda x: -x[2])[:n]:
    print(f"{x[0]:>22} {100 * x[2] / tot:5.1f}% {100 * x[3] / toti:5.1f}%  {x[1]}")
