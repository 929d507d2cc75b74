#!/usr/bin/env python
"""Probe k_greedy timing on a workload while varying the Alg. 2 budget and the launch shape.
Usage (GPU): python tools/probe_greedy.py [workload]"""
import itertools
import os
import subprocess
import sys
import json

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(wl_name, ns, rook, T, G):
    code = f"""
import sys, json
sys.path.insert(0, {ROOT!r})
import torch
from paper_1903_11554_b200 import TTCross
from workloads import WORKLOADS
wl = WORKLOADS[{wl_name!r}]
u, w = wl.grid()
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
tt = TTCross(wl.family, torch.from_numpy(u).cuda(), torch.from_numpy(w).cuda(), wl.rank_cap, wl.tol,
             n_samples={ns}, rook_iters={rook}, seed=wl.seed, stream=s.cuda_stream)
for _ in range(3):
    tt.solve_launch(wl.alg6_sweeps, graph=False); tt.integrate_read()
tt.set_timing(True)
tt.solve_launch(wl.alg6_sweeps, graph=False); tt.integrate_read()
kt = tt.kernel_times(); st = tt.stats()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
tt.set_timing(False)
ev[0].record(s)
for _ in range(10):
    tt.solve_launch(wl.alg6_sweeps, graph=True)
ev[1].record(s); torch.cuda.synchronize()
print(json.dumps(dict(greedy_us=kt['k_greedy'][1]*1e3/kt['k_greedy'][0], rook=st['rook_steps'],
      ext_us=kt['k_sb_extend'][1]*1e3/kt['k_sb_extend'][0], tab_us=kt['k_sb_tables'][1]*1e3/kt['k_sb_tables'][0],
      solve_ms=ev[0].elapsed_time(ev[1])/10)))
"""
    env = dict(os.environ, TTC_GREEDY_T=str(T), TTC_GREEDY_G=str(G))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    if out.returncode:
        return {"error": out.stderr[-300:]}
    return json.loads(out.stdout.strip().splitlines()[-1])


if __name__ == "__main__":
    wl = sys.argv[1] if len(sys.argv) > 1 else "D5"
    for (ns, rook), (T, G) in itertools.product([(32, 4), (32, 0), (1, 0), (32, 1)],
                                                 [(512, 16), (256, 16), (512, 8), (512, 4), (512, 1), (256, 1)]):
        r = one(wl, ns, rook, T, G)
        print(json.dumps({"wl": wl, "ns": ns, "rook": rook, "T": T, "G": G, **r}), flush=True)
