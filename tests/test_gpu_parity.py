"""GPU parity: the CUDA path (through the C-ABI) against the oracle on the same seeded inputs.

Bar (BASELINE.json north_star): pivot index sets bit-exact, fiber entries within 1e-13
relative (they are in fact compared bit-exactly, R3), integral within 1e-12
relative.  Small cases span several cluster tiles and ragged tails; the BASELINE configs
run at full size (C_4, D_5, C_10 whole; D_20 and C_200 on sampled interfaces of the first
half-sweep plus size-independent properties of the full run).
"""
import numpy as np
import pytest

from oracle import cross as X
from oracle import integrand as ig
from workloads import FAMILY_C, FAMILY_D, WORKLOADS, ising_grid

pytestmark = pytest.mark.gpu

INT_RTOL = 1e-12


def make(family, d, n, L, cap, tol, p, seed, delta=1e-2, max_swaps=0):
    from paper_1903_11554_b200 import TTCross
    u, w = ising_grid(d, n, L)
    tt = TTCross(family, u, w, cap, tol, n_enrich=p, max_swaps=max_swaps, delta=delta, seed=seed)
    prob = X.Problem(family, u, w, cap, tol, p, delta, max_swaps, seed)
    return tt, prob


def assert_same_state(tt, st, where=""):
    ranks, piv = tt.state()
    assert list(ranks) == st.ranks, f"ranks differ {where}: {list(ranks)} vs {st.ranks}"
    for i, (a, b) in enumerate(zip(piv, st.piv)):
        assert np.array_equal(a, b), f"pivots of interface {i} differ {where}"


def check_run(tt, prob, sweeps, check_fibers=True):
    st = X.initial_state(prob)
    assert_same_state(tt, st, "at init")
    for s in range(sweeps):
        for direction in (X.DIR_LR, X.DIR_RL):
            tt.half_sweep(direction)
            tt.commit()
            st = X.half_sweep(prob, st, direction)
            assert_same_state(tt, st, f"after sweep {s} dir {direction}")
        st.sweep += 1
    val, log10, sign = tt.integrate()
    fibers = X.tt_fibers(prob, st)
    _, _, _, nev = X.integrate(prob, st, fibers)
    ref, rlog10, rsign = X.integrate_exact(prob, st, fibers)
    if check_fibers:
        for m in range(prob.d):
            g = tt.fiber(m)
            assert g.shape == fibers[m].shape
            assert np.array_equal(g, fibers[m]), f"fiber {m} differs (max rel {np.max(np.abs(g - fibers[m]) / np.abs(fibers[m]).max()):.2e})"
    assert sign == rsign
    assert abs(log10 - rlog10) < 1e-12 * max(1.0, abs(rlog10))
    if np.isfinite(ref) and ref != 0:
        assert abs(val - ref) <= INT_RTOL * abs(ref), (val, ref)
    stats = tt.stats()
    assert stats["evals"] == st.n_evals + nev
    return st, val


@pytest.mark.parametrize("family,d,n,L,cap,tol,p,seed,sweeps", [
    (FAMILY_C, 2, 9, 3.0, 4, 1e-12, 2, 1, 2),          # single interface
    (FAMILY_C, 3, 5, 2.0, 8, 1e-12, 4, 2, 2),          # ranks limited by n^k
    (FAMILY_D, 3, 7, 3.0, 5, 1e-12, 3, 3, 2),
    (FAMILY_C, 4, 33, 8.0, 6, 1e-12, 3, 4, 3),
    (FAMILY_D, 5, 17, 6.0, 8, 1e-11, 4, 5, 3),
    (FAMILY_D, 6, 31, 6.0, 7, 1e-11, 2, 6, 2),         # ragged: odd n, odd cap
    (FAMILY_C, 7, 65, 10.0, 12, 1e-13, 5, 7, 2),
    (FAMILY_C, 3, 97, 12.0, 1, 1e-12, 0, 8, 2),        # rank 1, no enrichment
    (FAMILY_D, 4, 41, 8.0, 16, 0.0, 16, 9, 2),         # tol = 0, max enrichment
])
def test_parity_small(lib, family, d, n, L, cap, tol, p, seed, sweeps):
    tt, prob = make(family, d, n, L, cap, tol, p, seed)
    check_run(tt, prob, sweeps)
    tt.close()


def test_parity_max_rank_and_swap_cap(lib):
    tt, prob = make(FAMILY_C, 3, 129, 20.0, 64, 1e-15, 16, 10, max_swaps=3)
    check_run(tt, prob, 1)
    tt.close()


def test_reset_reproduces(lib):
    tt, prob = make(FAMILY_D, 4, 25, 6.0, 6, 1e-12, 3, 12)
    tt.sweep(2)
    v1 = tt.integrate()
    r1 = tt.state()
    tt.reset()
    tt.sweep(2)
    v2 = tt.integrate()
    r2 = tt.state()
    assert v1 == v2
    assert all(np.array_equal(a, b) for a, b in zip(r1[1], r2[1]))
    tt.close()


def test_zero_tensor_is_singular(lib):
    """D_3 on a 2-node grid vanishes identically (two coordinates always coincide):
    every fiber is zero, the pivots are kept (R8) and the quadrature reports a singular
    intersection, like the oracle's solve."""
    from paper_1903_11554_b200 import TTCError
    tt, prob = make(FAMILY_D, 3, 2, 1.0, 2, 1e-12, 1, 13)
    tt.sweep(1)
    st = X.sweep(prob, X.initial_state(prob))
    assert_same_state(tt, st)
    with pytest.raises(TTCError) as e:
        tt.integrate()
    assert "code 3" in str(e.value)
    with pytest.raises(np.linalg.LinAlgError):
        X.integrate(prob, st)
    tt.close()


def test_device_resident_inputs(lib):
    import torch
    from paper_1903_11554_b200 import TTCross
    u, w = ising_grid(4, 33, 8.0)
    tt_h = TTCross(FAMILY_C, u, w, 6, 1e-12, n_enrich=2, seed=3)
    tt_d = TTCross(FAMILY_C, torch.from_numpy(u).cuda(), torch.from_numpy(w).cuda(), 6, 1e-12, n_enrich=2, seed=3,
                   stream=torch.cuda.current_stream().cuda_stream)
    tt_h.sweep(2)
    tt_d.sweep(2)
    assert tt_h.integrate() == tt_d.integrate()
    tt_h.close()
    tt_d.close()


@pytest.mark.parametrize("name", ["C4", "D5", "C10"])
def test_parity_baseline_configs_full(lib, name):
    wl = WORKLOADS[name]
    tt, prob = make(wl.family, wl.d, wl.n, wl.L, wl.rank_cap, wl.tol, wl.n_enrich, wl.seed, wl.maxvol_delta,
                    wl.max_swaps)
    check_run(tt, prob, wl.sweeps, check_fibers=(name != "C10"))
    tt.close()


@pytest.mark.parametrize("name,ifaces", [("D20", [0, 9, 18]), ("C200", [0, 57, 198])])
def test_parity_large_configs_sampled(lib, name, ifaces):
    """Full-size configs: the first L->R half-sweep of sampled interfaces against the oracle
    (inputs are the seed-derived initial pivots, computed independently by the oracle)."""
    wl = WORKLOADS[name]
    tt, prob = make(wl.family, wl.d, wl.n, wl.L, wl.rank_cap, wl.tol, wl.n_enrich, wl.seed, wl.maxvol_delta,
                    wl.max_swaps)
    st0 = X.initial_state(prob)
    assert_same_state(tt, st0, "at init")
    tt.half_sweep(X.DIR_LR)
    tt.commit()
    ranks, piv = tt.state()
    for i in ifaces:
        new, info = X.update_interface(prob, st0, i, X.DIR_LR)
        assert np.array_equal(piv[i], new), f"{name}: interface {i} differs"
    tt.close()


@pytest.mark.parametrize("name", ["D20", "C200"])
def test_large_configs_properties(lib, name):
    """Size-independent properties of the full run: ranks within the cap, distinct left
    and right parts, nonsingular intersections (the quadrature succeeds), a finite integral
    and the evaluation count of the schedule."""
    wl = WORKLOADS[name]
    tt, prob = make(wl.family, wl.d, wl.n, wl.L, wl.rank_cap, wl.tol, wl.n_enrich, wl.seed, wl.maxvol_delta,
                    wl.max_swaps)
    tt.sweep(2)
    val, log10, sign = tt.integrate()
    assert sign == 1 and np.isfinite(log10)
    ranks, piv = tt.state()
    for i, P in enumerate(piv):
        assert 1 <= len(P) <= wl.rank_cap
        assert len({tuple(r[:i + 1]) for r in P}) == len(P)
        assert len({tuple(r[i + 1:]) for r in P}) == len(P)
        assert np.all((P >= 0) & (P < wl.n))
    # sampled fiber entries of the final quadrature pass equal the integrand at their indices
    rng = np.random.default_rng(0)
    for m in rng.choice(wl.d, 3, replace=False):
        F = tt.fiber(int(m))
        L = piv[m - 1] if m > 0 else np.zeros((1, wl.d), np.int64)
        R = piv[m] if m < wl.d - 1 else np.zeros((1, wl.d), np.int64)
        for _ in range(20):
            al, be, a = rng.integers(F.shape[0]), rng.integers(F.shape[1]), rng.integers(wl.n)
            idx = np.concatenate([L[al][:m], [a], R[be][m + 1:]])
            assert F[al, be, a] == ig.entries(wl.family, prob.u, idx[None, :])[0]
    tt.close()
