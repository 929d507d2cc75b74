#!/usr/bin/env python
"""Per-source-line stall samples of one kernel from an ncu report (diagnostics).

ncu's source page (SASS view, with the per-instruction "Warp Stall Sampling" columns) is
joined, by section offset, with the line table nvdisasm -g prints for the same cubin (compile
with -lineinfo).  Out-of-line subroutines live in the kernel's text section under
`$kernel$function` labels, so their samples are attributed to their own lines / function.

    python tools/ncu_lines.py <report.ncu-rep> <library.so> <kernel mangled name> [top] [--kernel REGEX]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def line_table(so, kernel):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True, check=True)
    cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    out = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout
    table, cur, curline, func = {}, False, None, kernel
    for ln in out.split("\n"):
        if ln.startswith(kernel + ":"):
            cur = True
            continue
        if cur and re.match(r"^_Z\w+:\s*$", ln):
            break
        if not cur:
            continue
        m = re.match(r"^\s*\$" + re.escape(kernel) + r"\$(\w+):", ln)
        if m:
            func = m.group(1)
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            curline = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            table[int(m.group(1), 16)] = (curline, func, m.group(2).strip())
    return table


def main():
    rep, so, kernel = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 and sys.argv[4].isdigit() else 40
    kf = ["-k", "regex:" + sys.argv[sys.argv.index("--kernel") + 1]] if "--kernel" in sys.argv else []
    csv_text = subprocess.run(["ncu", "-i", rep, *kf, "--page", "source", "--csv", "--print-source=sass"],
                              capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(csv_text)))
    hdr = rows[1]
    ia, iall, inot = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), \
        hdr.index("Warp Stall Sampling (Not-issued Samples)")
    iex = hdr.index("Instructions Executed")
    # per-reason stall columns, when the source page has them
    ireason = [(i, h) for i, h in enumerate(hdr) if ("stall" in h.lower() and "Sampling" not in h)]
    if "--headers" in sys.argv:
        print("# columns:", hdr)
    data = rows[2:]
    for i, r in enumerate(data):   # (a report may print the kernel's page more than once)
        if r and r[0] == "Kernel Name":
            data = data[:i]
            break
    base = int(data[0][ia], 16)
    table = line_table(so, kernel)
    by_line = collections.defaultdict(lambda: [0, 0, 0])
    by_func = collections.defaultdict(lambda: [0, 0, 0])
    by_line_reason = collections.defaultdict(collections.Counter)
    ffilter = sys.argv[sys.argv.index("--func") + 1] if "--func" in sys.argv else None
    by_fline = collections.defaultdict(lambda: [0, 0])
    tot = 0
    for r in data:
        off = int(r[ia], 16) - base
        s_all, s_not, ex = int(r[iall] or 0), int(r[inot] or 0), int(r[iex] or 0)
        tot += s_all
        line, func, _ = table.get(off, (None, "?", ""))
        by_line[line][0] += s_all
        by_line[line][1] += s_not
        by_line[line][2] += ex
        for i, h in ireason:
            try:
                by_line_reason[line][h] += float(r[i] or 0)
            except ValueError:
                pass
        by_func[func][0] += s_all
        by_func[func][1] += s_not
        by_func[func][2] += ex
        if ffilter and re.search(ffilter, func):
            by_fline[line][0] += s_all
            by_fline[line][1] += ex
    print(f"# {rep}: {tot} stall samples, {len(data)} instructions")
    print("## by function (samples, share, not-issued, warp instructions executed)")
    for f, v in sorted(by_func.items(), key=lambda kv: -kv[1][0]):
        print(f"{100 * v[0] / tot:6.1f}% {v[0]:9d} {v[1]:9d} {v[2]:12d}  {f[:90]}")
    if ffilter:
        print(f"## lines of functions matching {ffilter} (samples, share of all, warp instructions)")
        for ln, v in sorted(by_fline.items(), key=lambda kv: (str(kv[0][0]) if kv[0] else "", kv[0][1] if kv[0] else 0)):
            rs = by_line_reason.get(ln)
            top3 = ", ".join(f"{h.strip()} {int(c)}" for h, c in rs.most_common(4) if "Not Issued" not in h) if rs else ""
            print(f"{v[0]:9d} {100 * v[0] / tot:6.2f}% {v[1]:12d}  {ln}  {top3}")
    print(f"## top {top} lines")
    for ln, v in sorted(by_line.items(), key=lambda kv: -kv[1][0])[:top]:
        rs = by_line_reason.get(ln)
        top3 = ", ".join(f"{h.replace('Warp Stall Sampling','').strip()} {int(c)}" for h, c in rs.most_common(3)) if rs else ""
        print(f"{100 * v[0] / tot:6.1f}% {v[0]:9d} {v[2]:12d}  {ln}  {top3}")


if __name__ == "__main__":
    main()
