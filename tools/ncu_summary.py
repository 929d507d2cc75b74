#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel:
launches, total device time, share.  Usage: ncu_summary.py launches.csv [title]"""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}


def summarise(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("ttc::", "")
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
    return agg


if __name__ == "__main__":
    agg = summarise(sys.argv[1])
    tot = sum(v[1] for v in agg.values())
    print(f"# {sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]}")
    print(f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare shares)")
    print(f"{'kernel':40s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:40s} {v[0]:8d} {v[1]:12.1f} {v[1] / v[0]:10.2f} {100 * v[1] / tot:6.1f}%")
    print(f"{'TOTAL':40s} {sum(v[0] for v in agg.values()):8d} {tot:12.1f}")
