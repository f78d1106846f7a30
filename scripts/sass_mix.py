"""Opcode mix and hottest SASS lines of one kernel from `ncu --page source --print-source sass --csv`."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
nxt = [i for i, r in enumerate(rows) if i > 0 and r and r[0] == "Kernel Name"]
rows = rows[:nxt[0]] if nxt else rows   # (the page repeats the kernel block)
h = rows[1]
iA, iS, iI, iT = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
mix = collections.Counter(); tot = 0; lines = []
for r in rows[2:]:
    if len(r) < len(h): continue
    try: n = int(r[iI]); st = int(r[iT])
    except ValueError: continue
    src = r[iS].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"): op = src.split()[1]
    mix[op.split(".")[0]] += n; tot += n
    lines.append((n, st, r[iA][-5:], src))
print("total warp instructions", tot)
for op, n in mix.most_common(30): print(f"{op:10s} {n:12d} {100*n/tot:5.1f}%")
if len(sys.argv) > 2:
    for n, st, a, s in sorted(lines, key=lambda x: -x[0])[:int(sys.argv[2])]: print(f"{n:10d} {st:6d} {a} {s}")
