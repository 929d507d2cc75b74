#!/usr/bin/env python
"""Oracle goldens for the full-size BASELINE configs (D_20 = configs[3], C_200 = configs[4]).

Test infrastructure: imports only ``oracle/`` and ``workloads`` (no CUDA path).  The full
oracle solve of these configs takes CPU-hours on one core, so this script runs each sweep's
superblock updates in a process pool -- one task per superblock, each calling
``oracle.cross.sweep(prob, st, [k])`` on the state of the previous sweep (Alg. 6,
lines 624-641: every superblock reads only the previous sweep's index sets, so the pool order
cannot change the result; pinned by tests/test_oracle_cross.py::
test_parallel_partition_equals_all_at_once) -- and evaluates the quadrature fibers mode by
mode in the same pool.

Output ``tests/golden/<name>.npz``:
  piv    (d-1, cap, d) int32   final pivot tuples, -1 beyond the rank (slots never move,
                               Alg. 6 line 4, so the state after ANY sweep s is the first
                               ranks[s][k] slots of interface k)
  par    (d-1, cap, 2) int32   parents (alpha, beta) of those slots
  ranks  (sweeps+1, d-1) int32 ranks after 0, 1, ..., sweeps sweeps
  evals  (sweeps+1,)     int64 the oracle's evaluation counter after each sweep
  integral_exact  [value, log10|value|, sign]  oracle.cross.integrate_exact (R9) of the final
                                               cross (fp64 fibers, mpmath chain)
  integral_fp64   [value, log10|value|, sign]  oracle.cross.integrate (fp64 chain)
  meta   json string: workload parameters, sweep count, wall time

    python tools/make_goldens.py D20 C200 [--workers 7]
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import cross as X  # noqa: E402
from workloads import WORKLOADS  # noqa: E402

_PROB = None


def _init(name):
    global _PROB
    wl = WORKLOADS[name]
    u, w = wl.grid()
    _PROB = X.Problem(wl.family, u, w, wl.rank_cap, wl.tol, wl.n_samples, wl.rook_iters, wl.seed, wl.fold)


def _update(args):
    st, k = args
    new = X.sweep(_PROB, st, [k])
    info = new.log[-1][1][k]
    return k, new.piv[k], new.par[k], info["evals"]


def _fiber(args):
    st, m = args
    d = _PROB.d
    F = X.fiber(_PROB, st.piv[m - 1] if m > 0 else None, m, st.piv[m] if m < d - 1 else None)
    return m, F


def generate(name, workers, out_dir):
    wl = WORKLOADS[name]
    _init(name)
    prob = _PROB
    d, cap = prob.d, prob.rank_cap
    t0 = time.time()
    st = X.initial_state(prob)
    ranks = [list(st.ranks)]
    evals = [st.n_evals]
    with mp.get_context("fork").Pool(workers, initializer=_init, initargs=(name,)) as pool:
        for s in range(wl.alg6_sweeps):
            new = st.copy()
            order = sorted(range(d - 1), key=lambda k: -(st.ranks[k] * ((st.ranks[k - 1] if k else 1) +
                                                                          (st.ranks[k + 1] if k < d - 2 else 1))))
            for k, piv, par, ev in pool.imap_unordered(_update, [(st, k) for k in order]):
                new.piv[k], new.par[k] = piv, par
                new.n_evals += ev
            new.sweep = st.sweep + 1
            st = new
            ranks.append(list(st.ranks))
            evals.append(st.n_evals)
            print(f"{name} sweep {s + 1}/{wl.alg6_sweeps}: max rank {max(st.ranks)}, {time.time() - t0:.0f} s",
                  flush=True)
        fibers = [None] * d
        for m, F in pool.imap_unordered(_fiber, [(st, m) for m in range(d)]):
            fibers[m] = F
    print(f"{name}: fibers done, {time.time() - t0:.0f} s", flush=True)
    v64, l64, s64, _ = X.integrate(prob, st, fibers)
    vex, lex, sex = X.integrate_exact(prob, st, fibers)
    print(f"{name}: integral {vex!r} (log10 {lex!r}, sign {sex}), fp64 chain {v64!r}, {time.time() - t0:.0f} s",
          flush=True)
    piv = np.full((d - 1, cap, d), -1, np.int32)
    par = np.full((d - 1, cap, 2), -1, np.int32)
    for k in range(d - 1):
        r = len(st.piv[k])
        piv[k, :r] = st.piv[k]
        par[k, :r] = st.par[k]
    meta = {"workload": name, "family": wl.family, "d": d, "n": wl.n, "L": wl.L, "rank_cap": cap, "tol": wl.tol,
            "n_samples": wl.n_samples, "rook_iters": wl.rook_iters, "seed": wl.seed, "alg6_sweeps": wl.alg6_sweeps,
            "generator": "tools/make_goldens.py (oracle only)", "wall_s": round(time.time() - t0, 1),
            "workers": workers}
    path = os.path.join(out_dir, f"{name}.npz")
    np.savez_compressed(path, piv=piv, par=par, ranks=np.array(ranks, np.int32), evals=np.array(evals, np.int64),
                        integral_exact=np.array([vex, lex, sex], np.float64),
                        integral_fp64=np.array([v64, l64, s64], np.float64), meta=json.dumps(meta))
    print(f"wrote {path}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="+", choices=sorted(WORKLOADS))
    ap.add_argument("--workers", type=int, default=max(1, (os.cpu_count() or 2) - 1))
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden"))
    a = ap.parse_args()
    for name in a.names:
        generate(name, a.workers, a.out)


if __name__ == "__main__":
    main()
