#!/usr/bin/env python
"""Print the per-sweep phase log written by tools/probe_phases.py --log (us per sweep)."""
import json
import sys

KEYS = ["prologue", "tables", "extend", "ext_raw", "ext_rec", "ext_rows_cta", "ext_cols_cta", "samples", "rook", "col_eval", "col_argmax",
        "row_eval", "row_argmax", "final", "exit", "rounds"]
for path in sys.argv[1:]:
    rows = [json.loads(l) for l in open(path) if l.startswith("{")]
    for r in rows:
        if "phase_us_per_launch" in r:
            print(r["workload"], "job", r["job"], "k_sweep_us", round(r["k_sweep_us"]), r["shape"])
    lg = [r for r in rows if "sweep" in r]
    step = max(1, len(lg) // 16)
    print("  sw " + " ".join(f"{k[:7]:>7s}" for k in KEYS) + "   total")
    for r in lg[::step] + lg[-1:]:
        tot = sum(r[k] for k in ["prologue", "tables", "extend", "samples", "rook", "final", "exit"])
        print(f"{r['sweep']:4d} " + " ".join(f"{r.get(k, 0):7.1f}" for k in KEYS) + f" {tot:7.1f}")
