"""GPU parity: the CUDA path (through the C-ABI) against the oracle on the same seeded inputs.

Bar (BASELINE.json north_star): pivot index sets bit-exact, fiber entries within 1e-13
relative (they are in fact compared bit-exactly, R3), integral within 1e-12
relative of the oracle's near-exact §4.1 contraction.  Small cases span several cluster
CTAs and ragged tails; the BASELINE configs C_4, D_5 and C_10 run whole; D_20 and C_200 are
checked on their first sweeps (the oracle's cost grows like r^3 n d^2 per sweep) plus
size-independent properties of the full run.
"""
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

from oracle import cross as X
from oracle import integrand as ig
from workloads import FAMILY_C, FAMILY_D, WORKLOADS, ising_grid

pytestmark = pytest.mark.gpu

INT_RTOL = 1e-12


def make(family, d, n, L, cap, tol, ns, rook, seed):
    from paper_1903_11554_b200 import TTCross
    u, w = ising_grid(d, n, L)
    tt = TTCross(family, u, w, cap, tol, n_samples=ns, rook_iters=rook, seed=seed)
    prob = X.Problem(family, u, w, cap, tol, ns, rook, seed)
    return tt, prob


def make_wl(wl):
    return make(wl.family, wl.d, wl.n, wl.L, wl.rank_cap, wl.tol, wl.n_samples, wl.rook_iters, wl.seed)


def assert_same_state(tt, st, where=""):
    ranks, piv, par = tt.state(parents=True)
    assert list(ranks) == st.ranks, f"ranks differ {where}: {list(ranks)} vs {st.ranks}"
    for k in range(len(piv)):
        assert np.array_equal(piv[k], st.piv[k]), f"pivots of interface {k} differ {where}"
        assert np.array_equal(par[k], st.par[k]), f"parents of interface {k} differ {where}"


def gpu_sweep_evals(prob, before, after, prev_rows, prev_cols):
    """Entries the CUDA path evaluates in one sweep: u/v of the existing pivots on the rows /
    columns that are new since the previous sweep (the oracle recomputes them all), plus the
    oracle's own Alg. 2 search evaluations (samples + rook columns/rows)."""
    d, n = prob.d, prob.n
    total = 0
    rows_done, cols_done = [], []
    for k in range(d - 1):
        rl = before.ranks[k - 1] if k > 0 else 1
        rr = before.ranks[k + 1] if k < d - 2 else 1
        r = before.ranks[k]
        total += (rl - prev_rows[k]) * n * r + (rr - prev_cols[k]) * n * r
        total += after.log[-1][1][k]["search_evals"]
        rows_done.append(rl)
        cols_done.append(rr)
    return total, rows_done, cols_done


WSUM_RTOL = 1e-28


def assert_wsum_matches(got, F, w, m):
    """W_m = sum_a w_a F[:, :, a] (§4.1) from the fused fiber kernel in
    double-double against the oracle's double-double sum of the oracle's fibers: every term
    w_a A >= 0, so both are within ~n 2^-104 relative of the exact sum; bar 1e-28 relative."""
    hi, lo = got
    rh, rl = X._dd_weighted_sum(F, w)
    assert hi.shape == rh.shape, (m, hi.shape, rh.shape)
    diff = np.abs((hi - rh) + (lo - rl))
    bad = diff > WSUM_RTOL * np.abs(rh)
    assert not np.any(bad), f"W_{m}: {int(bad.sum())} entries beyond 1e-28, worst {np.max(diff / np.maximum(np.abs(rh), 1e-300))}"


def quad_evals(prob, st):
    d, n = prob.d, prob.n
    r = [1] + st.ranks + [1]
    return sum(r[m] * r[m + 1] * n for m in range(d)) + sum(x * x for x in st.ranks)


def check_run(tt, prob, sweeps, check_fibers=True, check_evals=True):
    st = X.initial_state(prob)
    assert_same_state(tt, st, "at init")
    expect = 0   # the rank-1 start (X.N_INIT evaluations) belongs to loading the grid
    prev_rows = [0] * (prob.d - 1)
    prev_cols = [0] * (prob.d - 1)
    for s in range(sweeps):
        tt.sweep(1)
        new = X.sweep(prob, st)
        assert_same_state(tt, new, f"after sweep {s}")
        e, prev_rows, prev_cols = gpu_sweep_evals(prob, st, new, prev_rows, prev_cols)
        expect += e
        st = new
    val, log10, sign = tt.integrate()
    fibers = X.tt_fibers(prob, st)
    ref, rlog10, rsign = X.integrate_exact(prob, st, fibers)
    if check_fibers:
        # the weighted sums the product kernel contracted (read before fiber() refreshes them)
        for m in range(prob.d):
            assert_wsum_matches(tt.wsum(m), fibers[m], prob.qw[m], m)
        for m in range(prob.d):
            g = tt.fiber(m)   # the entries of the same kernel (k_fiber_wsum, EMIT)
            assert g.shape == fibers[m].shape
            assert np.array_equal(g, fibers[m]), f"fiber {m} differs"
    assert sign == rsign
    assert abs(log10 - rlog10) < 1e-12 * max(1.0, abs(rlog10))
    if np.isfinite(ref) and ref != 0:
        assert abs(val - ref) <= INT_RTOL * abs(ref), (val, ref)
    if check_evals:
        assert tt.stats()["evals"] == expect + quad_evals(prob, st)
    return st, val


@pytest.mark.parametrize("family,d,n,L,cap,tol,ns,rook,seed,sweeps", [
    (FAMILY_C, 2, 9, 3.0, 4, 1e-12, 8, 4, 1, 5),          # a single superblock, no neighbours
    (FAMILY_C, 3, 5, 2.0, 8, 1e-12, 16, 4, 2, 9),         # ranks limited by the grid (tol stop)
    (FAMILY_D, 3, 7, 3.0, 5, 1e-12, 16, 4, 3, 6),
    (FAMILY_C, 4, 33, 8.0, 6, 1e-12, 32, 4, 4, 7),
    (FAMILY_D, 5, 17, 6.0, 8, 1e-11, 32, 4, 5, 8),
    (FAMILY_D, 6, 31, 6.0, 7, 1e-11, 7, 2, 6, 7),         # ragged: odd n, odd cap, odd samples
    (FAMILY_C, 7, 65, 10.0, 12, 1e-13, 64, 4, 7, 12),
    (FAMILY_C, 3, 97, 12.0, 1, 1e-12, 4, 4, 8, 3),        # rank cap 1: no additions ever
    (FAMILY_D, 4, 41, 8.0, 16, 0.0, 1024, 1, 9, 16),      # tol = 0, max samples, one rook round
    (FAMILY_C, 4, 21, 6.0, 6, 1e-12, 16, 0, 10, 6),       # no rook rounds: the best sample
    (FAMILY_D, 3, 513, 24.0, 64, 1e-12, 32, 4, 11, 4),    # cap*n = 32832 rows: 4-CTA clusters
    (FAMILY_D, 4, 65, 8.0, 24, 1e-14, 32, 4, 12, 24),     # ranks past one 16x16 fiber tile, ragged
    (FAMILY_C, 5, 129, 10.0, 40, 1e-15, 32, 4, 13, 40),   # ranks 40: three tiles, ragged last one
])
def test_parity_small(lib, family, d, n, L, cap, tol, ns, rook, seed, sweeps):
    tt, prob = make(family, d, n, L, cap, tol, ns, rook, seed)
    check_run(tt, prob, sweeps)
    tt.close()


def test_reset_and_graph_reproduce(lib):
    wl = WORKLOADS["C4"]
    tt, prob = make_wl(wl)
    tt.sweep(wl.alg6_sweeps)
    v1 = tt.integrate()
    s1 = tt.state(parents=True)
    tt.solve_launch(wl.alg6_sweeps, graph=True)
    v2 = tt.integrate_read()
    s2 = tt.state(parents=True)
    tt.solve_launch(wl.alg6_sweeps, graph=False)
    v3 = tt.integrate_read()
    tt.reset()
    tt.sweep(wl.alg6_sweeps)
    v4 = tt.integrate()
    assert v1 == v2 == v3 == v4
    for a, b in zip(s1[1] + s1[2], s2[1] + s2[2]):
        assert np.array_equal(a, b)
    tt.close()


def test_zero_tensor_is_singular(lib):
    """D_3 on a 2-node grid vanishes identically (two coordinates always coincide): the
    first pivot is zero, every superblock is left unchanged (R8) and the quadrature reports a
    singular intersection, like the oracle's solve."""
    from paper_1903_11554_b200 import TTCError
    tt, prob = make(FAMILY_D, 3, 2, 1.0, 2, 1e-12, 4, 4, 13)
    tt.sweep(2)
    st = X.sweep(prob, X.sweep(prob, X.initial_state(prob)))
    assert_same_state(tt, st)
    with pytest.raises(TTCError) as e:
        tt.integrate()
    assert "code 3" in str(e.value)
    with pytest.raises(np.linalg.LinAlgError):
        X.integrate(prob, st)
    tt.close()


def test_device_resident_inputs_and_load_grid(lib):
    import torch
    from paper_1903_11554_b200 import TTCross
    u, w = ising_grid(4, 33, 8.0)
    tt_h = TTCross(FAMILY_C, u, w, 6, 1e-12, n_samples=16, seed=3)
    tt_d = TTCross(FAMILY_C, torch.from_numpy(u).cuda(), torch.from_numpy(w).cuda(), 6, 1e-12, n_samples=16, seed=3,
                   stream=torch.cuda.current_stream().cuda_stream)
    tt_h.sweep(6)
    tt_d.sweep(6)
    ref = tt_h.integrate()
    assert ref == tt_d.integrate()
    # a different grid, then the original one again through tt_cross_load_grid
    u2, w2 = ising_grid(4, 33, 6.0)
    tt_d.load_grid(u2, w2)
    tt_d.sweep(6)
    other = tt_d.integrate()
    assert other != ref
    tt_d.load_grid(torch.from_numpy(u).pin_memory().numpy(), w)
    tt_d.solve_launch(6, graph=True)
    assert tt_d.integrate_read() == ref
    tt_h.close()
    tt_d.close()


@pytest.mark.parametrize("name", ["C4", "D5", "C10"])
def test_parity_baseline_configs_full(lib, name):
    wl = WORKLOADS[name]
    tt, prob = make_wl(wl)
    check_run(tt, prob, wl.alg6_sweeps, check_fibers=(name != "C10"))
    tt.close()


@pytest.mark.parametrize("name,sweeps", [("D20", 3), ("C200", 2)])
def test_parity_large_configs_first_sweeps(lib, name, sweeps):
    """Full-size configs: the first sweeps of the bench launch configuration against the
    oracle (pivots, parents, ranks bit-exact; eval counter)."""
    wl = WORKLOADS[name]
    tt, prob = make_wl(wl)
    st = X.initial_state(prob)
    assert_same_state(tt, st, "at init")
    for s in range(sweeps):
        tt.sweep(1)
        st = X.sweep(prob, st)
        assert_same_state(tt, st, f"after sweep {s}")
    tt.close()


@pytest.mark.parametrize("name", ["D20", "C200"])
def test_large_configs_properties(lib, name):
    """Size-independent properties of the full bench solve: ranks within the cap, nested and
    distinct index sets (eq. (4)), nonsingular intersections (the quadrature succeeds), a
    finite integral, and fiber entries equal to the integrand at their indices (sampled)."""
    wl = WORKLOADS[name]
    tt, prob = make_wl(wl)
    tt.solve_launch(wl.alg6_sweeps, graph=True)
    val, log10, sign = tt.integrate_read()
    assert sign != 0 and np.isfinite(log10)
    ranks, piv, par = tt.state(parents=True)
    assert 1 < max(ranks) <= wl.rank_cap   # C_200 stops below the cap on tol (values ~1e-9 of max)
    for k, P in enumerate(piv):
        assert 1 <= len(P) <= wl.rank_cap
        assert len({tuple(r[:k + 1]) for r in P}) == len(P)
        assert len({tuple(r[k + 1:]) for r in P}) == len(P)
        assert np.all((P >= 0) & (P < wl.n))
        for s, (al, be) in enumerate(par[k]):
            if k > 0:
                assert np.array_equal(P[s][:k], piv[k - 1][al][:k])
            if k < wl.d - 2:
                assert np.array_equal(P[s][k + 2:], piv[k + 1][be][k + 2:])
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


@pytest.mark.parametrize("family,d,n,L,cap,sweeps", [
    (FAMILY_C, 1000, 9, 4.0, 3, 2),      # d near the paper's largest (C_1024), C family
    (FAMILY_D, 24, 1024, 30.0, 4, 2),    # 276 pairs per entry; n >> d^2 so that seeded samples avoid A = 0
    (FAMILY_C, 3, 4096, 30.0, 2, 2),     # maximum n
    (FAMILY_C, 2, 64, 8.0, 64, 3),       # rank cap = grid size along the single interface
])
def test_parity_extreme_sizes(lib, family, d, n, L, cap, sweeps):
    """Size limits: pivots, parents and ranks bit-exact against the oracle after every sweep,
    eval counter, and a nonsingular quadrature."""
    tt, prob = make(family, d, n, L, cap, 1e-12, 8, 2, 17)
    check_run(tt, prob, sweeps, check_fibers=(d <= 40))
    tt.close()


@pytest.mark.parametrize("name,modes", [("D5", [0, 2, 4]), ("C10", [0, 5, 9]), ("D20", [1, 10, 19])])
def test_theorem1_interpolation_of_gpu_cross(lib, name, modes):
    """Theorem 1 on the CUDA path's own cross after the full bench
    solve: eq. (3) built from the returned fibers and the intersection matrices (entries
    from the oracle's integrand) reproduces sampled fiber entries A(I_{<=m-1}, i_m, I_{>m}).
    Holds because every sweep kept the index sets nested; relative tolerance scales with
    cond(M_k) (numpy fp64 solves)."""
    wl = WORKLOADS[name]
    tt, prob = make_wl(wl)
    tt.solve_launch(wl.alg6_sweeps, graph=True)
    tt.integrate_read()
    ranks, piv = tt.state()
    d = wl.d
    st = X.State(piv, [np.zeros((len(p), 2), np.int64) for p in piv])
    Ms = [X.intersection(prob, st, k) for k in range(d - 1)]
    Fs = {}

    def fib(m):
        if m not in Fs:
            Fs[m] = tt.fiber(m)
        return Fs[m]

    rng = np.random.default_rng(1)
    for m in modes:
        F = fib(m)
        for _ in range(3):
            al, be, a = rng.integers(F.shape[0]), rng.integers(F.shape[1]), rng.integers(wl.n)
            L = piv[m - 1][al] if m > 0 else None
            Rr = piv[m][be] if m < d - 1 else None
            idx = np.concatenate([L[:m] if L is not None else [], [a], Rr[m + 1:] if Rr is not None else []]).astype(int)
            # eq. (3) left to right: F_0[:, i_0, :] M_0^{-1} F_1[:, i_1, :] ... at idx
            v = fib(0)[0, :, idx[0]]
            for q in range(1, d):
                v = np.linalg.solve(Ms[q - 1].T, v)
                v = v @ fib(q)[:, :, idx[q]]
            exact = F[al, be, a]
            conds = max(np.linalg.cond(M) for M in Ms)
            assert abs(float(v[0]) - exact) <= max(1e-10, 1e-15 * conds * d) * max(abs(exact), 1e-300) \
                or abs(float(v[0]) - exact) <= 1e-13 * np.max(np.abs(F)), (m, float(v[0]), exact)
    tt.close()


def test_c_demo_matches_python_binding(lib):
    """The plain-C program (examples/ttcross_demo.c) and the Python binding give the same
    D_5 integral (one library, no Python in the C path).  The C program builds its u-nodes
    with libm's exp, numpy's exp may differ by an ulp on some nodes, hence a tolerance."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([os.path.join(root, "examples", "ttcross_demo")], capture_output=True, text=True,
                         timeout=120)
    assert out.returncode == 0, out.stderr
    c_val = float(out.stdout.split("D_5 = ")[1].split()[0])
    wl = WORKLOADS["D5"]
    tt, prob = make_wl(wl)
    tt.sweep(wl.alg6_sweeps)
    py_val = tt.integrate()[0]
    tt.close()
    assert abs(c_val - py_val) <= 1e-12 * abs(py_val), (c_val, py_val)


def test_perturbed_timing_same_pivots(lib):
    """Race detector: the step-trace build (thread 0 of every CTA delayed at every phase and
    rook-step boundary) must reproduce the product build's pivots exactly, run after run, on
    a cached (D_5) and an uncached 16-CTA-cluster (C_10) configuration.  This caught a read of
    the pivot value E(x*, y*) racing with its owner's in-place rescaling of V[r][:]."""
    import subprocess
    import sys
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "check_trace_build.py"), "C10", "D5"],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("name", ["D5", "C10"])
def test_fiber_kernel_cluster_splits_agree(lib, name, monkeypatch):
    """The quadrature fiber kernel splits each tile's nodes over a (1, NS, 1) cluster and adds
    the partial double-double sums through DSMEM in range order: every split (NS = 1, 2, 4, 8,
    forced with TTC_FW_NS) gives the same integral to double-double rounding, and the oracle's
    within the parity bar."""
    from paper_1903_11554_b200 import TTCross
    wl = WORKLOADS[name]
    u, w = wl.grid()
    prob = X.Problem(wl.family, u, w, wl.rank_cap, wl.tol, wl.n_samples, wl.rook_iters, wl.seed)
    st = X.initial_state(prob)
    for _ in range(wl.alg6_sweeps):
        st = X.sweep(prob, st)
    ref, *_ = X.integrate_exact(prob, st)
    vals = []
    for ns in ("1", "2", "4", "8"):
        monkeypatch.setenv("TTC_FW_NS", ns)
        tt = TTCross(wl.family, u, w, wl.rank_cap, wl.tol, n_samples=wl.n_samples, rook_iters=wl.rook_iters,
                     seed=wl.seed)
        tt.sweep(wl.alg6_sweeps)
        vals.append(tt.integrate()[0])
        tt.close()
    for v in vals:
        assert abs(v - vals[0]) <= 1e-14 * abs(vals[0]), vals
        assert abs(v - ref) <= INT_RTOL * abs(ref), (v, ref)
