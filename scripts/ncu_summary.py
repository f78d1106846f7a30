#!/usr/bin/env python
"""Summarise ncu captures into profiles/ (tracked): one JSON + markdown per round.

  python scripts/ncu_summary.py --tag r01 --full gpurun_out/match_r01.ncu-rep \
      --launches gpurun_out/launches_r01.csv [--config C5] [--update-traffic]

--full   : a `ncu --set full` capture of the top kernel (one launch)
--launches: the `--metrics gpu__time_duration.sum` launch list of a bench run
--update-traffic writes profiles/traffic.json (read by bench.py for roofline.traffic)
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RAW_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_bytes.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for i, h in enumerate(hdr):
            if h in RAW_METRICS or h in ("Kernel Name",):
                d[h] = (r[i], units[i])
        res.append(d)
    return res


def to_num(v, unit):
    try:
        x = float(str(v).replace(",", ""))
    except ValueError:
        return v
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
             "byte": 1.0, "Kbyte": 1e3,
             "Mbyte": 1e6, "Gbyte": 1e9}.get(unit)
    return x * scale if scale else x


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        us = to_num(d["Metric Value"], d["Metric Unit"])
        name = d["Kernel Name"].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
        agg.setdefault(name, []).append(us)
    return {k: {"n": len(v), "mean_us": sum(v) / len(v), "total_us": sum(v)} for k, v in agg.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--full")
    ap.add_argument("--launches")
    ap.add_argument("--config", default="C5")
    ap.add_argument("--update-traffic", action="store_true")
    args = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    summary = {"tag": args.tag, "config": args.config}
    md = [f"# ncu summary {args.tag} ({args.config})", ""]
    if args.full:
        ks = raw(args.full)
        summary["full"] = []
        for k in ks:
            e = {m: to_num(*k[m]) for m in k if m != "Kernel Name"}
            e["kernel"] = k["Kernel Name"][0]
            e["dram_bytes"] = (e.get("dram__bytes_read.sum", 0) or 0) + (e.get("dram__bytes_write.sum", 0) or 0)
            summary["full"].append(e)
            md.append(f"## {e['kernel']}")
            md += [f"- {m}: {e[m]}" for m in RAW_METRICS if m in e]
            md.append(f"- dram bytes (read+write): {e['dram_bytes']:.0f}")
            md.append("")
        if args.update_traffic and summary["full"]:
            tpath = os.path.join(ROOT, "profiles", "traffic.json")
            t = json.load(open(tpath)) if os.path.exists(tpath) else {}
            # the capture holds one launch of each match-stage kernel (k_project, k_match)
            t.setdefault("match_stage", {})[args.config] = sum(e["dram_bytes"] for e in summary["full"])
            t.setdefault("per_kernel", {})[args.config] = {e["kernel"].split("(")[0]: e["dram_bytes"]
                                                           for e in summary["full"]}
            t["source"] = f"ncu --set full capture {args.tag}"
            json.dump(t, open(tpath, "w"), indent=1)
    if args.launches:
        la = launches(args.launches)
        summary["launches"] = la
        tot = sum(v["total_us"] for v in la.values())
        md += ["## launch list (ncu gpu__time_duration, cold-cache, serialised)", "",
               "| kernel | launches | mean us | share |", "|---|---|---|---|"]
        for k, v in sorted(la.items(), key=lambda kv: -kv[1]["total_us"]):
            md.append(f"| {k} | {v['n']} | {v['mean_us']:.1f} | {v['total_us'] / tot * 100:.1f}% |")
    json.dump(summary, open(os.path.join(ROOT, "profiles", f"ncu_{args.tag}.json"), "w"), indent=1)
    open(os.path.join(ROOT, "profiles", f"ncu_{args.tag}.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
