#!/usr/bin/env python
"""Per-phase device time of k_sweep (globaltimer, CTA 0 of one superblock: the middle one
unless TTC_PHASE_JOB is set; "prologue" = the neighbour wait of the persistent kernel).
Usage (GPU): python tools/probe_phases.py D5 C10 ..."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if not os.environ.get("TTC_LIB_PATH"):   # the phase clocks live in a diagnostics build
    import __graft_entry__  # noqa: E402
    os.environ["TTC_LIB_PATH"] = __graft_entry__.build_diagnostics()

import torch  # noqa: E402

from paper_1903_11554_b200 import TTCross  # noqa: E402
from workloads import WORKLOADS  # noqa: E402

for name in [a for a in sys.argv[1:] if not a.startswith("--")] or ["D5"]:
    wl = WORKLOADS[name]
    job = int(os.environ.get("TTC_PHASE_JOB", (wl.d - 1) // 2))
    os.environ["TTC_PHASE_JOB"] = str(job)
    u, w = wl.grid()
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    tt = TTCross(wl.family, torch.from_numpy(u).cuda(), torch.from_numpy(w).cuda(), wl.rank_cap, wl.tol,
                 n_samples=wl.n_samples, rook_iters=wl.rook_iters, seed=wl.seed, stream=s.cuda_stream)
    for _ in range(3):
        tt.solve_launch(wl.alg6_sweeps, graph=True)
        tt.integrate_read()
    tt.set_timing(True)
    tt.solve_launch(wl.alg6_sweeps, graph=False)
    tt.integrate_read()
    ph, log = tt.phase_times(per_sweep=True)
    kt = tt.kernel_times()
    tt.set_timing(False)
    nl = max(1.0, ph.pop("launches"))
    per = {k: round(v / nl, 2) for k, v in ph.items()}
    print(json.dumps({"workload": name, "job": job, "shape": tt.launch_shape(), "k_sweep_us": kt["k_sweep"][1] * 1e3 / kt["k_sweep"][0],
                      "phase_us_per_launch": per, "rook_steps": tt.stats()["rook_steps"]}), flush=True)
    if "--log" in sys.argv:
        for s, row in enumerate(log):
            print(json.dumps({"workload": name, "job": job, "sweep": s, **row}), flush=True)
    tt.close()
    os.environ.pop("TTC_PHASE_JOB")
