#!/usr/bin/env python3
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of bench.py.

usage: tools/launch_summary.py <launches.csv> [steps]
Prints per kernel: launches, total ms, ms per launch, and the share of the last `steps`
solves (the timed region: everything after the last k_fp64_peak / warm-up solves is
attributed by taking the trailing launches that belong to `steps` solves, delimited by
k_scan_input, which opens every solve).  ncu times are cold-cache and serialised; compare
shares, not absolute times, with bench.py's live CUDA-event numbers.
"""
import collections
import csv
import re
import sys


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"^void ", "", name)
    return name.replace("mr3::", "")


def main(path, steps=1):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.reader(lines)
    h = next(rd)
    ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    for r in rd:
        if r[mi] == "gpu__time_duration.sum":
            rows.append((short(r[ki]), float(r[vi].replace(",", "")) * 1e-6))  # ns -> ms
    starts = [i for i, (k, _) in enumerate(rows) if k.startswith("k_scan_input")]
    timed = rows[starts[-steps]:] if len(starts) >= steps else rows
    agg = collections.OrderedDict()
    for k, ms in timed:
        base = re.sub(r"<.*", "", k)
        c, t = agg.get(base, (0, 0.0))
        agg[base] = (c + 1, t + ms)
    tot = sum(t for _, t in agg.values())
    print(f"{'kernel':28s} {'launches':>8s} {'ms':>10s} {'ms/launch':>10s} {'share':>7s}")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:28s} {c:8d} {t:10.3f} {t / c:10.4f} {100 * t / tot:6.1f}%")
    print(f"{'total (timed solves)':28s} {sum(c for c, _ in agg.values()):8d} {tot:10.3f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
