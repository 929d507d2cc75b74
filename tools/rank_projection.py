#!/usr/bin/env python
"""Per-rank compute of the partitioned (multi-GPU) path on ONE GPU, as a projection of the
P-GPU solve time (diagnostics; this pool has one GPU).

The P rank contexts (world = P) of a workload run their tt_cross_sweep_local one after the
other on the same device -- each rank's kernel has the whole GPU to itself, as it would on its
own GPU; nothing waits on another launch -- with the all-gather of Alg. 6 lines 6-8 emulated by
device copies (tests/test_gpu_multirank.py).  Per sweep the projected time is the slowest
rank's k_sweep device time (tt_cross_set_timing) plus an assumed all-gather latency; the
quadrature adds the slowest rank's local contraction.  Prints one JSON line per (workload, P).
Usage (GPU): python tools/rank_projection.py D20 C200 [--allgather-us 15]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from paper_1903_11554_b200 import TTCross  # noqa: E402
from workloads import WORKLOADS  # noqa: E402
from test_gpu_multirank import exchange  # noqa: E402

ag_us = float(sys.argv[sys.argv.index("--allgather-us") + 1]) if "--allgather-us" in sys.argv else 15.0
names = [a for a in sys.argv[1:] if a in WORKLOADS] or ["D20"]
for name in names:
    wl = WORKLOADS[name]
    u, w = wl.grid()
    for P in (1, 2, 4, 8):
        tts = [TTCross(wl.family, u, w, wl.rank_cap, wl.tol, n_samples=wl.n_samples, rook_iters=wl.rook_iters,
                       seed=wl.seed, rank=p, world=P) for p in range(P)]
        xv = [t.exchange_view() for t in tts]
        per = xv[0][1] // 4
        shapes = [t.launch_shape() for t in tts]
        sweep_ms = []
        prev = [0.0] * P   # (kernel_times accumulates since the context's last reset)
        for t in tts:
            t.set_timing(True)
        for s in range(wl.alg6_sweeps):
            ms = []
            for p, t in enumerate(tts):
                t.sweep_local()
                torch.cuda.synchronize()
                cur = t.kernel_times()["k_sweep"][1]
                ms.append(cur - prev[p])
                prev[p] = cur
            sweep_ms.append(max(ms))
            if P > 1:
                exchange([v for v, _ in xv], per)
            for t in tts:
                t.commit()
        q = []
        for t in tts:
            before = sum(v[1] for k, v in t.kernel_times().items() if k != "k_sweep")
            t.integrate_local()
            torch.cuda.synchronize()
            q.append(sum(v[1] for k, v in t.kernel_times().items() if k != "k_sweep") - before)
            t.set_timing(False)
        if P > 1:
            pv = [t.partials_view() for t in tts]
            exchange([v for v, _ in pv], pv[0][1] // 8)
        val = tts[0].integrate_finish()
        for t in tts:
            t.close()
        total = sum(sweep_ms) + (len(sweep_ms) * ag_us / 1e3 if P > 1 else 0.0) + max(q)
        print(json.dumps({"workload": name, "P": P, "projected_ms": round(total, 3),
                          "sweeps_ms": round(sum(sweep_ms), 3), "quadrature_ms": round(max(q), 3),
                          "allgather_us_assumed": ag_us if P > 1 else 0, "integral": val[0],
                          "rank0_shape": shapes[0], "superblocks_rank0": None}), flush=True)
