#!/usr/bin/env python
"""Local-memory accesses (LDL/STL) inside loops of a function's SASS (diagnostics): a spill in a
hot loop of the sweep kernel costs an L2 round trip under the factor stream.

    python tools/sass_loop_spills.py <cubin|so> <function-name-substring | =exact-name> [kernel-substring]

Loops = [target, branch] ranges of backward branches.  Prints each loop's size and its LDL/STL
count, and the LDL/STL outside loops."""
import os
import re
import subprocess
import sys
import tempfile


def sass_of(path):
    if path.endswith(".so"):
        tmp = tempfile.mkdtemp()
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(path)], cwd=tmp, capture_output=True, check=True)
        path = os.path.join(tmp, [f for f in os.listdir(tmp) if f.endswith(".cubin")][0])
    return subprocess.run(["nvdisasm", "-c", path], capture_output=True, text=True).stdout


def main():
    path, fn = sys.argv[1], sys.argv[2]
    kern = sys.argv[3] if len(sys.argv) > 3 else None
    out = sass_of(path).split("\n")
    # function bodies: a label line ending in ':' that names the function (possibly $kernel$fn)
    body, on = [], False
    for ln in out:
        m = re.match(r"^(\S+):\s*$", ln)
        if m and not ln.startswith(".L") and not ln.startswith(".text"):
            name = m.group(1)
            on = (name == fn[1:]) if fn.startswith('=') else (fn in name and (kern is None or kern in name))
            if on:
                body.append(("LABEL", name))
            continue
        if on:
            body.append(("I", ln))
    ins = []   # (addr, text)
    labels = {}
    for kind, ln in body:
        if kind == "LABEL":
            print("function:", ln)
            continue
        m = re.match(r"^(\.L_x_\d+):", ln.strip())
        if m:
            labels[m.group(1)] = len(ins)
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            ins.append((int(m.group(1), 16), m.group(2)))
    loops = []
    for i, (a, t) in enumerate(ins):
        m = re.search(r"BRA\s.*`\((\.L_x_\d+)\)", t)
        if m and m.group(1) in labels and labels[m.group(1)] <= i:
            loops.append((labels[m.group(1)], i))
    inloop = [False] * len(ins)
    for b, e in loops:
        for i in range(b, e + 1):
            inloop[i] = True
    tot_in = tot_out = 0
    for b, e in sorted(loops):
        n = sum(1 for i in range(b, e + 1) if re.search(r"\b(LDL|STL)\b", ins[i][1]))
        if n:
            print(f"loop {ins[b][0]:#x}-{ins[e][0]:#x}: {e - b + 1} instructions, {n} LDL/STL")
    for i, (a, t) in enumerate(ins):
        if re.search(r"\b(LDL|STL)\b", t):
            if inloop[i]:
                tot_in += 1
            else:
                tot_out += 1
    print(f"{len(ins)} instructions, {len(loops)} loops; LDL/STL inside loops {tot_in}, outside {tot_out}")


if __name__ == "__main__":
    main()
