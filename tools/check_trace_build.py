#!/usr/bin/env python
"""Race detector: the -DTTC_TRACE build (tools/trace_steps.py) slows thread 0 of every CTA at
each phase / step boundary by a global read-modify-write, which shifts the interleaving of the
sweep kernels' CTAs and clusters.  Both builds must give the same pivots, run after run.
Exit status 1 on any difference.  Usage (GPU): python tools/check_trace_build.py C10 D5 ..."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from paper_1903_11554_b200 import binding  # noqa: E402
from workloads import WORKLOADS  # noqa: E402


def run(lib_path, name, reps, sweeps=None):
    binding._lib = None
    binding.load(lib_path)
    from paper_1903_11554_b200 import TTCross
    wl = WORKLOADS[name]
    u, w = wl.grid()
    out = []
    for _ in range(reps):
        tt = TTCross(wl.family, u, w, wl.rank_cap, wl.tol, n_samples=wl.n_samples, rook_iters=wl.rook_iters,
                     seed=wl.seed)
        tt.sweep(sweeps or wl.alg6_sweeps)
        ranks, piv = tt.state()
        out.append((list(ranks), [p.copy() for p in piv]))
        tt.close()
    return out


def same(a, b):
    return a[0] == b[0] and all(np.array_equal(x, y) for x, y in zip(a[1], b[1]))


import trace_steps  # noqa: E402

trace_steps.build()
bad = 0
for name in sys.argv[1:] or ["C10"]:
    prod = run(binding.LIB_PATH, name, 5)
    trace = run(os.path.join(ROOT, "tools", "libttcross_trace.so"), name, 5)
    print(name, "prod deterministic", all(same(prod[0], p) for p in prod),
          "trace deterministic", all(same(trace[0], p) for p in trace),
          "trace==prod", [same(prod[0], t) for t in trace], "ranks", prod[0][0], trace[0][0], flush=True)
    ok = all(same(prod[0], p) for p in prod + trace)
    bad += not ok
    if not ok:
        for s in range(1, WORKLOADS[name].alg6_sweeps + 1):
            a = run(binding.LIB_PATH, name, 1, s)[0]
            b = run(os.path.join(ROOT, "tools", "libttcross_trace.so"), name, 1, s)[0]
            if not same(a, b):
                print("first difference after sweep", s, a[0], b[0])
                for k, (x, y) in enumerate(zip(a[1], b[1])):
                    if not np.array_equal(x, y):
                        print(" interface", k, "\n", x[-3:], "\n", y[-3:])
                break
sys.exit(1 if bad else 0)
