"""GPU parity at full size: the BASELINE configs D_20 (configs[3]) and C_200 (configs[4]) solved
whole by the CUDA path and compared with the oracle's full solve, plus small cases forced onto
the streamed rook-step path.

The oracle's full solves take CPU-hours, so they are stored: tests/golden/{D20,C200}.npz,
written by tools/make_goldens.py, which imports only oracle/ and workloads/ (ranks after every
sweep, the final pivots and parents -- slots never move, Alg. 6 line 4, so the state
after any sweep is a prefix of the final one -- and oracle.cross.integrate_exact of the final
cross).  The bar (BASELINE.json north_star): pivots and parents bit-exact after every Alg. 6
sweep, the integral within 1e-12 relative, W_m within 1e-28.

These solves run the non-cached launch shape whose column/row steps stream the u/v factors
through the shared-memory ring; the stats counter ring_steps proves it ran.
"""
import json
import os

import numpy as np
import pytest

from oracle import cross as X
from workloads import FAMILY_C, FAMILY_D, WORKLOADS, ising_grid

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
INT_RTOL = 1e-12


def load_golden(name):
    path = os.path.join(GOLDEN, f"{name}.npz")
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: run tools/make_goldens.py {name}")
    g = np.load(path)
    meta = json.loads(str(g["meta"]))
    wl = WORKLOADS[name]
    assert (meta["d"], meta["n"], meta["rank_cap"], meta["seed"], meta["alg6_sweeps"]) == \
        (wl.d, wl.n, wl.rank_cap, wl.seed, wl.alg6_sweeps), "golden was generated for another config"
    return g


def golden_state(g, s):
    """(ranks, [PIV[k]], [PAR[k]]) after sweep s (prefix of the final slots)."""
    ranks = [int(r) for r in g["ranks"][s]]
    piv = [g["piv"][k, :r].astype(np.int64) for k, r in enumerate(ranks)]
    par = [g["par"][k, :r].astype(np.int64) for k, r in enumerate(ranks)]
    return ranks, piv, par


def assert_state(tt, g, s):
    ranks, piv, par = tt.state(parents=True)
    granks, gpiv, gpar = golden_state(g, s)
    assert list(ranks) == granks, f"ranks after sweep {s}: {list(ranks)} vs {granks}"
    for k in range(len(piv)):
        assert np.array_equal(piv[k], gpiv[k]), f"pivots of interface {k} differ after sweep {s}"
        assert np.array_equal(par[k], gpar[k]), f"parents of interface {k} differ after sweep {s}"


def make_tt(wl, u, w):
    from paper_1903_11554_b200 import TTCross
    return TTCross(wl.family, u, w, wl.rank_cap, wl.tol, n_samples=wl.n_samples, rook_iters=wl.rook_iters,
                   seed=wl.seed)


@pytest.mark.parametrize("name", ["D20", "C200"])
def test_full_solve_sweep_by_sweep(lib, name):
    """Every Alg. 6 sweep of the full-size config, one launch per sweep, against the oracle."""
    g = load_golden(name)
    wl = WORKLOADS[name]
    u, w = wl.grid()
    tt = make_tt(wl, u, w)
    assert not tt.launch_shape()["cached"]
    assert_state(tt, g, 0)
    for s in range(wl.alg6_sweeps):
        tt.sweep(1)
        assert_state(tt, g, s + 1)
    assert tt.stats()["ring_steps"] > 0, "the streamed rook-step path did not run"
    tt.close()


@pytest.mark.parametrize("name", ["D20", "C200"])
def test_full_solve_bench_launch(lib, name):
    """The bench's launch configuration (one graph-replayed solve: persistent sweep kernel +
    quadrature): final pivots bit-exact, integral within 1e-12 of the oracle's near-exact
    contraction (R9), log10|I| likewise (C_200's grid sum is below the fp64 range of 4/d!)."""
    g = load_golden(name)
    wl = WORKLOADS[name]
    u, w = wl.grid()
    tt = make_tt(wl, u, w)
    tt.solve_launch(wl.alg6_sweeps, graph=True)
    val, log10, sign = tt.integrate_read()
    assert_state(tt, g, wl.alg6_sweeps)
    rval, rlog10, rsign = (float(x) for x in g["integral_exact"])
    assert sign == int(rsign)
    assert abs(log10 - rlog10) <= 1e-12 * max(1.0, abs(rlog10)) + 5e-13, (log10, rlog10)
    if rval != 0.0 and np.isfinite(rval):
        assert abs(val - rval) <= INT_RTOL * abs(rval), (val, rval)
    st = tt.stats()
    assert st["ring_steps"] > 0
    tt.close()


@pytest.mark.parametrize("name,modes", [("D20", [0, 10, 19]), ("C200", [0, 100, 199])])
def test_full_solve_wsum_entries(lib, name, modes):
    """The fused quadrature kernel's weighted sums W_m of the full-size cross against the
    oracle's double-double sums of the oracle's fibers on the golden index sets."""
    from test_gpu_parity import assert_wsum_matches
    g = load_golden(name)
    wl = WORKLOADS[name]
    u, w = wl.grid()
    tt = make_tt(wl, u, w)
    tt.solve_launch(wl.alg6_sweeps, graph=True)
    tt.integrate_read()
    prob = X.Problem(wl.family, u, w, wl.rank_cap, wl.tol, wl.n_samples, wl.rook_iters, wl.seed)
    _, piv, _ = golden_state(g, wl.alg6_sweeps)
    for m in modes:
        F = X.fiber(prob, piv[m - 1] if m > 0 else None, m, piv[m] if m < wl.d - 1 else None)
        assert_wsum_matches(tt.wsum(m), F, w[m], m)
        got = tt.fiber(m)
        assert np.array_equal(got, F), f"fiber {m} differs"
    tt.close()


@pytest.mark.parametrize("family,d,n,L,cap,sweeps", [
    (FAMILY_D, 5, 513, 24.0, 16, 16),
    (FAMILY_C, 6, 513, 20.0, 14, 14),
])
def test_streamed_rook_steps_small(lib, monkeypatch, family, d, n, L, cap, sweeps):
    """A case the oracle finishes in seconds, forced onto the streamed launch shape: one CTA
    per superblock (TTC_GREEDY_G=1, 256 threads), so a CTA owns r_{k-1} n >= 4 * 256 rows once
    the neighbour ranks reach 2 and its column/row steps stream the u/v factors through the
    shared-memory ring.  Pivots bit-exact after every sweep, fibers, W and the integral."""
    from test_gpu_parity import check_run, make
    monkeypatch.setenv("TTC_GREEDY_G", "1")
    monkeypatch.setenv("TTC_GREEDY_T", "256")
    tt, prob = make(family, d, n, L, cap, 1e-13, 32, 4, 21)
    shape = tt.launch_shape()
    assert shape["cluster"] == 1 and shape["threads"] == 256 and not shape["cached"]
    check_run(tt, prob, sweeps)
    assert tt.stats()["ring_steps"] > 0, "the streamed rook-step path did not run"
    tt.close()
