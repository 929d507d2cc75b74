"""GPU parity of the x-form families (eq. (9)-(11), the paper's own Gauss-Legendre
setup): pivots and fibers bit-exact against the oracle, the integral within 1e-12 of the
oracle's near-exact contraction, and D_8 against the value PAPER.md Fig. 5 prints."""
import json
import os

import numpy as np
import pytest

from oracle import cross as X
from workloads import FAMILY_CX, FAMILY_DX, FAMILY_EX, X_WORKLOADS, xform_grid

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def run_pair(family, d, n, cap, sweeps, ns=16, rook=4, seed=5, tol=1e-14, fold=False):
    from paper_1903_11554_b200 import TTCross
    x, w = xform_grid(d, n)
    tt = TTCross(family, x, w, cap, tol, n_samples=ns, rook_iters=rook, seed=seed, fold_weights=fold)
    prob = X.Problem(family, x, w, cap, tol, ns, rook, seed, fold)
    st = X.initial_state(prob)
    for s in range(sweeps):
        tt.sweep(1)
        st = X.sweep(prob, st)
        ranks, piv, par = tt.state(parents=True)
        assert list(ranks) == st.ranks, f"sweep {s}"
        for k in range(len(piv)):
            assert np.array_equal(piv[k], st.piv[k]) and np.array_equal(par[k], st.par[k]), f"sweep {s} k {k}"
    val, log10, sign = tt.integrate()
    fibers = X.tt_fibers(prob, st)
    for m in range(len(fibers)):
        assert np.array_equal(tt.fiber(m), fibers[m]), f"fiber {m}"
    ref, _, _ = X.integrate_exact(prob, st, fibers)
    assert abs(val - ref) <= 1e-12 * abs(ref), (val, ref)
    tt.close()
    return val


@pytest.mark.parametrize("family,d,n,cap,sweeps", [
    (FAMILY_CX, 4, 17, 8, 8), (FAMILY_DX, 5, 17, 8, 8), (FAMILY_EX, 4, 13, 6, 6),
    (FAMILY_CX, 12, 9, 6, 6), (FAMILY_DX, 3, 33, 16, 16),
])
def test_xform_parity(lib, family, d, n, cap, sweeps):
    run_pair(family, d, n, cap, sweeps)


def test_xform_d8_against_paper(lib):
    wl = X_WORKLOADS["Dx8"]
    val = run_pair(wl.family, wl.d, wl.n, wl.rank_cap, wl.sweeps, wl.n_samples, wl.rook_iters, wl.seed, wl.tol)
    ref = float(json.load(open(os.path.join(GOLD, "paper_values.json")))["D"]["8"])
    assert abs(val - ref) < 1e-9 * ref, (val, ref)


@pytest.mark.parametrize("family,d,n,cap,sweeps", [(FAMILY_CX, 5, 17, 8, 8), (FAMILY_DX, 6, 13, 8, 8)])
def test_xform_folded_parity(lib, family, d, n, cap, sweeps):
    """Weights folded into the tensor (§4.1): bit-exact as well."""
    run_pair(family, d, n, cap, sweeps, fold=True)


def test_xform_d8_folded_against_paper(lib):
    """Folding converges faster: rank 24 reaches ~4e-12 of the printed
    D_8 (unfolded: ~2e-11)."""
    wl = X_WORKLOADS["Dx8f"]
    val = run_pair(wl.family, wl.d, wl.n, wl.rank_cap, wl.sweeps, wl.n_samples, wl.rook_iters, wl.seed, wl.tol,
                   fold=True)
    ref = float(json.load(open(os.path.join(GOLD, "paper_values.json")))["D"]["8"])
    assert abs(val - ref) < 2e-11 * ref, (val, ref)
