"""The shared input generator: grids are exact, symmetric and match BASELINE.json."""
import json
import math
import os

import numpy as np

from workloads import WORKLOADS, ising_grid, trapezoid_t_grid

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_trapezoid_grid_exact_and_symmetric():
    for n, L in [(129, 20.0), (257, 20.0), (513, 24.0)]:
        t, w = trapezoid_t_grid(n, L)
        h = 2 * L / (n - 1)
        assert h == math.ldexp(math.frexp(h)[0], math.frexp(h)[1])  # representable
        assert np.array_equal(t, -t[::-1])                           # exact symmetry
        assert t[0] == -L and t[-1] == L
        assert abs(w.sum() - 2 * L) < 1e-12 and w[0] == h / 2
        u, _ = ising_grid(3, n, L)
        assert u.shape == (3, n) and np.all(u > 0)


def test_workloads_match_baseline_configs():
    cfg = json.load(open(os.path.join(ROOT, "BASELINE.json")))["configs"]
    assert len(cfg) == len(WORKLOADS)
    for text, wl in zip(cfg, WORKLOADS.values()):
        fam = "C" if wl.family == 0 else "D"
        assert f"{fam}_{wl.d} " in text
        assert f"{wl.n}-point" in text
        assert f"rank cap {wl.rank_cap}" in text
        assert f"[−{int(wl.L)},{int(wl.L)}]" in text


def test_alg6_sweeps_reach_the_cap_in_the_configured_sweeps():
    for wl in WORKLOADS.values():
        per = wl.alg6_sweeps // wl.sweeps
        assert wl.alg6_sweeps % wl.sweeps == 0
        assert 1 + wl.alg6_sweeps >= wl.rank_cap
        assert 1 + (per - 1) * wl.sweeps < wl.rank_cap or per == 1
