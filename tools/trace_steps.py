#!/usr/bin/env python
"""Step trace of the persistent sweep kernel (diagnostics, not part of the product).

Builds tools/libttcross_trace.so (the library with -DTTC_TRACE: thread 0 of every CTA appends
(point, clock64) events at the phase and rook-step boundaries of ttc_greedy.cuh), runs one
solve of each named workload and prints, per superblock, where the time of a sweep goes:
  tables / extend / cache+samples / rook steps (staging, evaluation incl. the CTA reduce,
  cluster barrier wait, DSMEM reduce) / final / neighbour wait.
Usage: python tools/trace_steps.py [--build] [--heavy] D5 C10 ...   (the run needs a GPU)
The default (light) variant buffers the events in shared memory; --heavy uses the race-detector
variant of tools/check_trace_build.py.
"""
import ctypes
import json
import os
import subprocess
import sys
from collections import defaultdict

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
MHZ = 1965.0   # SM clock under load on this pool's B200s (bench.py "clocks"): cycles -> us
LIB = os.path.join(ROOT, "tools", "libttcross_trace.so")          # heavy: race detector
LIB_LIGHT = os.path.join(ROOT, "tools", "libttcross_tracel.so")   # light: timing


def build(force=False, light=False):
    """compile a trace variant if it is missing or older than the sources"""
    import __graft_entry__ as g
    lib = LIB_LIGHT if light else LIB
    srcs = g._sources() + [os.path.join(ROOT, "include", "ttcross.h")]
    if not force and os.path.exists(lib) and all(os.path.getmtime(s) <= os.path.getmtime(lib) for s in srcs):
        return lib
    cmd = [g.NVCC, *g.NVCC_FLAGS, "-DTTC_TRACE=%d" % (2 if light else 1), "-o", lib,
           os.path.join(g.CSRC, "ttc_api.cu")]
    subprocess.run(cmd, check=True)
    return lib


POINT = {1: "start", 2: "tables_done", 3: "tables_sync", 4: "extend_done", 5: "extend_sync", 6: "cache",
         7: "samples_eval", 8: "rook_done", 9: "final_sync", 10: "col_begin", 11: "col_staged",
         20: "row_begin", 21: "row_staged", 31: "cta_reduced", 32: "published", 33: "cluster_wait",
         34: "step_end", 35: "red_read", 36: "red_reduced", 37: "expect_tx", 40: "end", 41: "end_sync", 49: "loop", 50: "nbr_waited", 51: "nbr_sync"}


def analyse(ev, cnt, G, njobs):
    """per-CTA event lists -> mean durations (us) per category, per job"""
    out = {}
    for job in range(njobs):
        acc = defaultdict(float)
        nst = defaultdict(int)
        for cr in range(G):
            b = job * G + cr
            m = min(int(cnt[b]), ev.shape[1])
            pts = (ev[b, :m] >> np.uint64(56)).astype(int)
            ts = (ev[b, :m] & np.uint64((1 << 56) - 1)).astype(np.int64)
            for i in range(1, m):
                a, z = pts[i - 1], pts[i]
                dt = (ts[i] - ts[i - 1]) / MHZ
                key = f"{POINT.get(a, a)}->{POINT.get(z, z)}"
                acc[key] += dt / G
                nst[key] += 1
        out[job] = {k: round(v, 2) for k, v in sorted(acc.items(), key=lambda kv: -kv[1])}
    return out


def per_sweep(ev, cnt, G, job, sweeps):
    """CTA 0 of `job`: one row per sweep, us from the sweep's loop point (49) to each phase
    boundary: nbr wait, tables, extension, samples, rook search, final, and the column/row
    steps (count, us)."""
    b = job * G
    m = min(int(cnt[b]), ev.shape[1])
    pts = (ev[b, :m] >> np.uint64(56)).astype(int)
    ts = (ev[b, :m] & np.uint64((1 << 56) - 1)).astype(np.int64)
    rows, cur = [], None
    for i in range(m):
        p, t = pts[i], ts[i]
        if p == 49:
            if cur:
                rows.append(cur)
            cur = {"t0": t, "marks": {}, "steps": 0, "step_us": 0.0, "last_step": None}
        elif cur is not None:
            cur["marks"].setdefault(p, t)
            if p in (10, 20):
                cur["last_step"] = t
            elif p == 34 and cur["last_step"] is not None:
                cur["steps"] += 1
                cur["step_us"] += (t - cur["last_step"]) / MHZ
                cur["last_step"] = None
    if cur:
        rows.append(cur)
    out = []
    for s, r in enumerate(rows):
        mk = r["marks"]
        def at(p):
            return (mk[p] - r["t0"]) / MHZ if p in mk else None
        out.append({"sweep": s, "wait": at(51), "tables": at(3), "extend": at(5), "samples": at(7),
                    "rook": at(8), "final": at(9), "end": at(40), "steps": r["steps"],
                    "step_us": round(r["step_us"], 1)})
    return out


def main():
    args = sys.argv[1:]
    light = "--heavy" not in args
    lib_path = build(force="--build" in args, light=light)
    args = [a for a in args if a not in ("--build", "--heavy")]
    import torch
    from paper_1903_11554_b200 import binding
    binding._lib = None
    lib = binding.load(lib_path)
    lib.ttc_trace_read.restype = ctypes.c_int
    from paper_1903_11554_b200 import TTCross
    from workloads import WORKLOADS
    slots, nev = 1024, 8192
    ev = np.zeros((slots, nev), dtype=np.uint64)
    cnt = np.zeros(slots, dtype=np.int32)
    for name in args or ["D5"]:
        wl = WORKLOADS[name]
        u, w = wl.grid()
        tt = TTCross(wl.family, u, w, wl.rank_cap, wl.tol, n_samples=wl.n_samples, rook_iters=wl.rook_iters,
                     seed=wl.seed)
        for _ in range(2):
            tt.solve_launch(wl.alg6_sweeps, graph=False)
            tt.integrate_read()
        lib.ttc_trace_read(ev.ctypes.data_as(ctypes.c_void_p), cnt.ctypes.data_as(ctypes.c_void_p))
        tt.solve_launch(wl.alg6_sweeps, graph=False)
        tt.integrate_read()
        torch.cuda.synchronize()
        lib.ttc_trace_read(ev.ctypes.data_as(ctypes.c_void_p), cnt.ctypes.data_as(ctypes.c_void_p))
        shape = tt.launch_shape()
        G = shape["cluster"]
        njobs = wl.d - 1
        res = analyse(ev, cnt, G, min(njobs, slots // G))
        total = {}
        for job in res:
            b = job * G
            m = min(int(cnt[b]), nev)
            ts = (ev[b, :m] & np.uint64((1 << 56) - 1)).astype(np.int64)
            total[job] = round((ts[-1] - ts[0]) / MHZ, 1) if m else 0
        print(json.dumps({"workload": name, "shape": shape, "events_cta0": int(cnt[0]), "span_us": total,
                          "per_job_us": {j: dict(list(v.items())[:24]) for j, v in res.items() if j < 4}}),
              flush=True)
        for job in sorted({0, njobs // 2, njobs - 1}):
            for row in per_sweep(ev, cnt, G, job, wl.alg6_sweeps):
                print(json.dumps({"workload": name, "job": job,
                                  **{k: (round(v, 1) if isinstance(v, float) else v) for k, v in row.items()}}),
                      flush=True)
        tt.close()


if __name__ == "__main__":
    main()
