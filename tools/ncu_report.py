#!/usr/bin/env python
"""Text summary of one `ncu --set full` capture (the sections judged under profiles/):
speed-of-light, scheduler and warp-state sections, launch shape, the warp-stall breakdown
from the source page and the per-launch DRAM traffic.  Also appends the traffic to
profiles/ncu_traffic.json under --key, which bench.py reads for its roofline "traffic".
Usage: ncu_report.py capture.ncu-rep title [--key WORKLOAD --out profiles/NAME.txt] [--kernel REGEX]
(needs only the ncu CLI; the summary goes to stdout, --out names it in ncu_traffic.json)"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SECTIONS = ["GPU Speed Of Light Throughput", "Compute Workload Analysis", "Memory Workload Analysis",
            "Scheduler Statistics", "Warp State Statistics", "Launch Statistics", "Occupancy"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "launch__registers_per_thread",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


KFILTER = []


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *KFILTER, *args, "--csv"], capture_output=True, text=True,
                         check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep, title = sys.argv[1], sys.argv[2]
    if "--kernel" in sys.argv:   # (a capture of several kernels: the one whose name matches)
        KFILTER.extend(["-k", "regex:" + sys.argv[sys.argv.index("--kernel") + 1]])
    key = sys.argv[sys.argv.index("--key") + 1] if "--key" in sys.argv else None
    rows = ncu_csv(rep, "--page", "details")
    h = rows[0]
    kname = rows[1][h.index("Kernel Name")]
    print(f"# {title}")
    print(f"# kernel: {kname}")
    for sec in SECTIONS:
        print(f"## {sec}")
        for r in rows[1:]:
            if r[h.index("Section Name")] == sec and r[h.index("Metric Name")]:
                print(f"  {r[h.index('Metric Name')]}: {r[h.index('Metric Value')]} {r[h.index('Metric Unit')]}")
    # stall reasons from the source page (pc sampling)
    src = ncu_csv(rep, "--page", "source", "--print-source=sass")
    hdr = next(r for r in src if r and r[0] == "Address")
    cols = [i for i, x in enumerate(hdr) if x.startswith("stall_") and "Not Issued" not in x]
    tot = collections.Counter()
    for r in src:
        if r and r[0].startswith("0x") and len(r) == len(hdr):
            for i in cols:
                if r[i].isdigit():
                    tot[hdr[i]] += int(r[i])
    s = sum(tot.values()) or 1
    print("## stall reasons (pc sampling, all warps)")
    for k, v in tot.most_common(12):
        print(f"  {k[6:]}: {100 * v / s:.1f}%")
    raw = ncu_csv(rep, "--page", "raw")
    rh, ru, rv = raw[0], raw[1], raw[2]
    vals = {}
    print("## raw (per launch)")
    for name in RAW:
        i = rh.index(name)
        print(f"  {name}: {rv[i]} {ru[i]}")
        vals[name] = float(rv[i].replace(",", "")) * SCALE.get(ru[i], 1.0)
    traffic = vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
    print(f"  traffic (read + write): {traffic:.6g} bytes")
    if key:
        path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        db = json.load(open(path)) if os.path.exists(path) else {}
        db[key] = {"kernel": kname.split("(")[0].replace("void ", ""), "dram_bytes_per_launch": traffic,
                   "source": sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else title}
        with open(path, "w") as f:
            json.dump(db, f, indent=1, sort_keys=True)
            f.write("\n")


if __name__ == "__main__":
    main()
