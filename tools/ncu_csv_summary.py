#!/usr/bin/env python3
"""Summarise an ncu --set full capture exported as CSV (tools/gpu_prof3.sh):
key metrics from the raw page, stall reasons, and the SASS opcode mix.

usage: tools/ncu_csv_summary.py <prefix>   (reads <prefix>_raw.csv and <prefix>_sass.csv[.gz])
"""
import csv
import gzip
import os
import sys
from collections import Counter

pre = sys.argv[1]
rows = list(csv.reader(open(pre + "_raw.csv")))
h = rows[0]
d = dict(zip(h, rows[2]))
units = dict(zip(h, rows[1]))
name = d.get("Kernel Name", "?")
print(f"== {name}")
keys = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "sm__warps_active.avg.per_cycle_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "local_load_bytes", "sass__inst_executed_local_loads"]
for k in keys:
    if k in d:
        print(f"   {k:70s} {d[k]} {units.get(k, '')}")
st = [(k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
       float(v)) for k, v in d.items()
      if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
      and v not in ("", "n/a")]
st.sort(key=lambda x: -x[1])
print("   stalls per issue: " + ", ".join(f"{k}={v:.2f}" for k, v in st[:8]))
sp = pre + "_sass.csv"
if not os.path.exists(sp) and os.path.exists(sp + ".gz"):
    sp += ".gz"
if os.path.exists(sp):
    op = gzip.open(sp, "rt") if sp.endswith(".gz") else open(sp)
    rows = list(csv.reader(op))
    h = rows[1]
    idx = {k: i for i, k in enumerate(h)}
    byop = Counter()
    for r in rows[2:]:
        src = r[idx["Source"]].strip()
        if not src:
            continue
        t = src.split()
        o = t[1] if t[0].startswith("@") else t[0]
        try:
            byop[o.split(".")[0]] += float(r[idx["Instructions Executed"]])
        except ValueError:
            pass
    tot = sum(byop.values())
    print(f"   SASS warp instructions executed: {tot:.4g}")
    print("   opcode mix: " + ", ".join(f"{k} {v / tot:.3f}" for k, v in byop.most_common(14)))
