#!/usr/bin/env python
"""Run whole solves of a workload through the product library (for ncu captures):
python tools/one_solve.py D5 [n_solves]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1903_11554_b200 import TTCross  # noqa: E402
from workloads import WORKLOADS  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "D5"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
u, w = wl.grid()
tt = TTCross(wl.family, u, w, wl.rank_cap, wl.tol, n_samples=wl.n_samples, rook_iters=wl.rook_iters, seed=wl.seed)
for _ in range(reps):
    tt.solve_launch(wl.alg6_sweeps, graph=False)
    print(tt.integrate_read())
tt.close()
