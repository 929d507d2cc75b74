"""Pins of oracle/cross.py against things other than itself (CPU only).

What fixes each expectation: the published splitmix64 test vector; explicit loops for the
first pivot; nestedness (eq. (4)); numpy.linalg solves of the cross formula
eq. (1) (independent arithmetic) for the error of every added pivot and for the rook
condition eq. (2); Theorem 1 (interpolation on nested crosses) and Theorem 2 (exact
recovery of exact-rank tensors); the TT formula eq. (3) evaluated entry by entry against
the full-grid sum for the §4.1 contraction; closed forms / brute force for the integral.
"""
import itertools

import numpy as np
import pytest

from oracle import cross as X
from oracle import integrand as ig
from workloads import FAMILY_C, FAMILY_D, ising_grid


def make_problem(fam, d, n, L, cap, tol=1e-12, ns=16, rook=4, seed=7):
    u, w = ising_grid(d, n, L)
    return X.Problem(fam, u, w, cap, tol, ns, rook, seed)


# ---------------------------------------------------------------- counter-based RNG
def test_splitmix64_reference_vector():
    # splitmix64 from state 0 (Steele, Lea, Flood 2014; the JDK SplittableRandom mixer):
    # first outputs are the published test vector below.
    ref = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F, 0xF88BB8A8724C81EC]
    assert [X.splitmix64(0, c) for c in range(4)] == ref


# ---------------------------------------------------------------- first pivot
@pytest.mark.parametrize("fam,d,n", [(FAMILY_C, 2, 5), (FAMILY_D, 4, 9), (FAMILY_D, 7, 33)])
def test_initial_state_is_argmax_of_seeded_samples(fam, d, n):
    prob = make_problem(fam, d, n, 4.0, 8)
    st = X.initial_state(prob)
    best, bv = None, -1.0
    for q in range(X.N_INIT):
        t = [X.splitmix64(prob.seed, ((0 * (d + 1) + 0) << 20) + q * d + j) % n for j in range(d)]
        v = abs(ig.entries(fam, prob.u, np.array([t]))[0])
        if v > bv:
            best, bv = t, v
    assert st.ranks == [1] * (d - 1)
    for k in range(d - 1):
        assert list(st.piv[k][0]) == best
        assert list(st.par[k][0]) == [0, 0]


# ---------------------------------------------------------------- superblock update
def superblock_dense(prob, st, k):
    sb = X.Superblock(prob, st, k)
    xs, ys = np.meshgrid(np.arange(sb.R), np.arange(sb.C), indexing="ij")
    return sb, prob.A(sb.tuples(xs, ys))


def cross_error(Asb, I, J):
    """E = A - A(:, J) A(I, J)^{-1} A(I, :)  (eq. (1)), via numpy.linalg.solve."""
    if not I:
        return Asb.copy()
    return Asb - Asb[:, J] @ np.linalg.solve(Asb[np.ix_(I, J)], Asb[I, :])


@pytest.mark.parametrize("fam,d,n,cap,rook", [(FAMILY_C, 3, 9, 6, 4), (FAMILY_D, 4, 7, 5, 4),
                                              (FAMILY_D, 3, 11, 8, 1), (FAMILY_C, 2, 13, 6, 0)])
def test_added_pivots_follow_alg2(fam, d, n, cap, rook):
    """Every added pivot's value is the cross error E(x*, y*) of the cross before it (eq. (1),
    computed with numpy.linalg, not the oracle's ACA updates); a converged rook search ends
    on an entry that dominates its row and column of |E| (eq. (2)); pivots are never
    removed; the tolerance test uses the largest |A| at the pivots."""
    prob = make_problem(fam, d, n, 3.0, cap, rook=rook)
    st = X.initial_state(prob)
    for sweep in range(7):
        new = X.sweep(prob, st)
        for k in range(d - 1):
            info = new.log[-1][1][k]
            sb, Asb = superblock_dense(prob, st, k)
            scale = np.max(np.abs(Asb))
            for add in info["adds"]:
                E = cross_error(Asb, add["xs_before"], add["ys_before"])
                E[add["xs_before"], :] = 0.0
                E[:, add["ys_before"]] = 0.0
                x, y = add["x"], add["y"]
                assert abs(add["pivot"] - E[x, y]) <= 1e-9 * scale
                if add["converged"]:
                    assert abs(E[x, y]) >= np.max(np.abs(E[:, y])) - 1e-9 * scale
                    assert abs(E[x, y]) >= np.max(np.abs(E[x, :])) - 1e-9 * scale
            assert np.array_equal(new.piv[k][:st.ranks[k]], st.piv[k])   # append-only (Alg. 6 line 4)
            assert new.ranks[k] <= cap
        st = new


@pytest.mark.parametrize("fam,d,n,cap,ns,rook", [(FAMILY_C, 3, 9, 6, 16, 4), (FAMILY_D, 4, 7, 5, 24, 0),
                                                 (FAMILY_D, 3, 11, 8, 8, 1), (FAMILY_C, 4, 6, 6, 40, 2)])
def test_search_starts_at_largest_sample_error(fam, d, n, cap, ns, rook):
    """Alg. 2 line 1: the rook search starts at the sample with the
    largest cross error |E| among the n_samples random superblock entries, pivot rows and
    columns excluded (E vanishes there).  The samples are
    re-drawn here from the counter-based stream (splitmix64, pinned by its published vector)
    and E is the numpy.linalg cross error of eq. (1), not the oracle's incomplete-LU factors.
    With rook = 0 the start is the added pivot itself."""
    prob = make_problem(fam, d, n, 3.0, cap, ns=ns, rook=rook)
    st = X.initial_state(prob)
    checked = 0
    for sweep in range(6):
        new = X.sweep(prob, st)
        for k in range(d - 1):
            info = new.log[-1][1][k]
            sb, Asb = superblock_dense(prob, st, k)
            scale = np.max(np.abs(Asb))
            R, C = Asb.shape
            for add in info["adds"]:
                tag = 1 + sweep
                sx = [X.splitmix64(prob.seed, ((tag * (d + 1) + k) << 20) + 2 * q) % R for q in range(ns)]
                sy = [X.splitmix64(prob.seed, ((tag * (d + 1) + k) << 20) + 2 * q + 1) % C for q in range(ns)]
                I, J = add["xs_before"], add["ys_before"]
                E = cross_error(Asb, I, J)
                e = np.array([0.0 if (x in I or y in J) else abs(E[x, y]) for x, y in zip(sx, sy)])
                x0, y0 = add["start"]
                q0 = next(q for q in range(ns) if (sx[q], sy[q]) == (x0, y0))
                assert e[q0] >= e.max() - 1e-9 * scale          # a largest |E| sample (up to rounding)
                if e.max() > 1e-6 * scale:
                    assert x0 not in I and y0 not in J          # pivot rows / columns excluded
                if rook == 0:
                    assert (add["x"], add["y"]) == (x0, y0)
                checked += 1
        st = new
    assert checked >= 3


def test_aca_form_equals_cross_formula():
    """The u/v factors rebuilt by the LU init reproduce A(:, J) A(I, J)^{-1} A(I, :)."""
    prob = make_problem(FAMILY_D, 4, 9, 3.0, 6)
    st = X.initial_state(prob)
    for _ in range(5):
        st = X.sweep(prob, st)
    k = 1
    sb, Asb = superblock_dense(prob, st, k)
    n = prob.n
    I = list(st.par[k][:, 0] * n + st.piv[k][:, k])
    J = list(st.par[k][:, 1] * n + st.piv[k][:, k + 1])
    approx = Asb[:, J] @ np.linalg.solve(Asb[np.ix_(I, J)], Asb[I, :])
    # interpolation property of the matrix cross: exact on its rows and columns
    assert np.max(np.abs(approx[I, :] - Asb[I, :])) <= 1e-10 * np.max(np.abs(Asb))
    assert np.max(np.abs(approx[:, J] - Asb[:, J])) <= 1e-10 * np.max(np.abs(Asb))


def test_tolerance_stops_exact_rank_superblock():
    """A rank-2 tensor: additions stop once the error is below tol (Alg. 2 with tol)."""
    u, w = ising_grid(4, 7, 2.0)
    prob = ExactRankProblem(FAMILY_C, u, w, 8, 1e-11, 16, 4, 5)
    st = X.initial_state(prob)
    for _ in range(4):
        st = X.sweep(prob, st)
    assert max(st.ranks) == 2
    for k in range(3):
        assert st.log[-1][1][k]["stop"] in ("tol", "cap", "n_add")


@pytest.mark.parametrize("d,n,cap", [(3, 5, 8), (5, 7, 6), (6, 4, 5)])
def test_sweeps_keep_nestedness_and_distinctness(d, n, cap):
    prob = make_problem(FAMILY_D, d, n, 3.0, cap)
    st = X.initial_state(prob)
    for _ in range(6):
        st = X.sweep(prob, st)
        for k, P in enumerate(st.piv):
            assert len({tuple(r[:k + 1]) for r in P}) == len(P) == len({tuple(r[k + 1:]) for r in P})
            assert np.all((P >= 0) & (P < n))
            for s, (al, be) in enumerate(st.par[k]):
                if k > 0:   # I_{<=k} subset of I_{<=k-1} x [n]   (eq. (4)), via the parent slot
                    assert np.array_equal(P[s][:k], st.piv[k - 1][al][:k])
                if k < d - 2:   # I_{>k} subset of [n] x I_{>k+1}
                    assert np.array_equal(P[s][k + 2:], st.piv[k + 1][be][k + 2:])


def test_parallel_partition_equals_all_at_once():
    """Alg. 6: updating disjoint superblock chunks separately and merging equals one sweep
    over all superblocks (each superblock only reads the previous state)."""
    prob = make_problem(FAMILY_C, 7, 9, 4.0, 5)
    st = X.sweep(prob, X.initial_state(prob))
    full = X.sweep(prob, st)
    merged = st.copy()
    for chunk in ([0, 1], [2, 3, 4], [5]):
        part = X.sweep(prob, st, chunk)
        for i in chunk:
            merged.piv[i], merged.par[i] = part.piv[i], part.par[i]
    for a, b in zip(full.piv, merged.piv):
        assert np.array_equal(a, b)


def test_eval_count_formula():
    """Entries evaluated per superblock = LU init r(R + C) + per addition: samples +
    (R + C) per rook round + the final column/row when the rook search did not end on them
    (the GPU path's counter is compared with the same per-sweep totals)."""
    prob = make_problem(FAMILY_C, 5, 9, 3.0, 7, ns=8, rook=2)
    st = X.sweep(prob, X.sweep(prob, X.initial_state(prob)))
    new = X.sweep(prob, st)
    total = 0
    for k in range(4):
        info = new.log[-1][1][k]
        R = (st.ranks[k - 1] if k > 0 else 1) * 9
        C = (st.ranks[k + 1] if k < 3 else 1) * 9
        assert info["evals"] >= st.ranks[k] * (R + C) + info["added"] * prob.n_samples
        total += info["evals"]
    assert new.n_evals - st.n_evals == total


# ---------------------------------------------------------------- TT formula / quadrature
def tt_entry(prob, st, idx):
    """Eq. (3): A~(i) = F_0[i_0] M_0^{-1} F_1[:, i_1, :] M_1^{-1} ... F_{d-1}[:, i_{d-1}]."""
    d = prob.d
    Fs = X.tt_fibers(prob, st)
    v = Fs[0][0, :, idx[0]]
    for m in range(1, d):
        M = X.intersection(prob, st, m - 1)
        v = v @ np.linalg.inv(M)
        v = v @ Fs[m][:, :, idx[m]]
    return float(v[0])


class AsymProblem(X.Problem):
    """A generic (non-symmetric, full-rank) smooth tensor for the cross identities."""

    def A(self, idx):
        U = np.stack([self.u[j][idx[..., j]] for j in range(self.d)], axis=-1)
        return 1.0 / (1.0 + np.sum(U * (1.0 + np.arange(self.d)), axis=-1))


def test_interpolation_theorem1_after_parallel_sweeps():
    """Theorem 1: the crosses produced by dimension-parallel sweeps
    stay nested, so eq. (3) interpolates every fiber entry A(I_{<=m-1}, i_m, I_{>m})."""
    u, w = ising_grid(4, 6, 3.0)
    prob = AsymProblem(FAMILY_C, u, w, 4, 1e-12, 8, 4, 7)
    st = X.initial_state(prob)
    for _ in range(4):
        st = X.sweep(prob, st)
    assert max(st.ranks) > 1
    for m in range(4):
        Lt = st.piv[m - 1] if m > 0 else np.zeros((1, 4), np.int64)
        Rt = st.piv[m] if m < 3 else np.zeros((1, 4), np.int64)
        for al in range(len(Lt)):
            for be in range(len(Rt)):
                for a in range(6):
                    idx = list(Lt[al][:m]) + [a] + list(Rt[be][m + 1:])
                    exact = prob.A(np.array([idx]))[0]
                    assert abs(tt_entry(prob, st, idx) - exact) <= 1e-9 * exact


def brute_tt_integral(prob, st):
    d, n = prob.d, prob.n
    tot = 0.0
    for idx in itertools.product(range(n), repeat=d):
        w = np.prod([prob.w[j][idx[j]] for j in range(d)])
        tot += w * tt_entry(prob, st, idx)
    return tot * ig.prefactor(d)


def test_integrate_equals_full_sum_of_tt_reconstruction():
    """§4.1 (lines 689-693): the (2d-1)-matrix product equals the quadrature of A~."""
    prob = make_problem(FAMILY_D, 3, 6, 3.0, 4)
    st = X.initial_state(prob)
    for _ in range(3):
        st = X.sweep(prob, st)
    val, log10, sign, _ = X.integrate(prob, st)
    ref = brute_tt_integral(prob, st)
    assert abs(val - ref) <= 1e-11 * abs(ref)


class ExactRankProblem(X.Problem):
    """A tensor of exact TT ranks <= 2: A(i) = sum_{s=1,2} prod_j g_s(u_{j,i_j})."""

    def A(self, idx):
        U = np.stack([self.u[j][idx[..., j]] for j in range(self.d)], axis=-1)
        return np.prod(1.0 / (1.0 + U), axis=-1) + np.prod(np.exp(-0.1 * U), axis=-1)


def test_exact_recovery_theorem2():
    """Theorem 2 (lines 344-350): exact-rank tensors are recovered exactly."""
    u, w = ising_grid(4, 7, 2.0)
    prob = ExactRankProblem(FAMILY_C, u, w, 4, 1e-11, 16, 4, 5)
    st = X.initial_state(prob)
    for _ in range(4):
        st = X.sweep(prob, st)
    assert max(st.ranks) == 2  # additions stop at the exact rank
    val, *_ = X.integrate(prob, st)
    d, n = 4, 7
    tot = 0.0
    for idx in itertools.product(range(n), repeat=d):
        wt = np.prod([w[j][idx[j]] for j in range(d)])
        tot += wt * prob.A(np.array([idx]))[0]
    assert abs(val - tot * ig.prefactor(d)) <= 1e-12 * abs(val)


def test_c4_converges_toward_brute_force():
    """Sanity of the whole pipeline: C_4 at rank cap 16 approaches the full-grid sum."""
    prob = make_problem(FAMILY_C, 4, 33, 8.0, 20, tol=1e-13, ns=32)
    st, val, _ = X.run(prob, 20)
    ref = ig.brute_force(FAMILY_C, prob.u, prob.w)
    assert abs(val - ref) < 1e-7 * ref


def test_integrate_exact_agrees_with_fp64_when_well_conditioned():
    """R9: the near-exact contraction equals the fp64 one to rounding on a well-conditioned
    cross, and equals the full-grid sum of the TT reconstruction (eq. (3))."""
    prob = make_problem(FAMILY_D, 3, 6, 3.0, 4)
    st = X.initial_state(prob)
    for _ in range(3):
        st = X.sweep(prob, st)
    v64, l64, s64, _ = X.integrate(prob, st)
    vex, lex, sex = X.integrate_exact(prob, st)
    assert s64 == sex and abs(v64 - vex) <= 1e-13 * abs(vex)
    assert abs(vex - brute_tt_integral(prob, st)) <= 1e-11 * abs(vex)


def test_dd_weighted_sum_is_accurate():
    import mpmath
    rng = np.random.default_rng(5)
    F = rng.standard_normal((3, 4, 200)) * np.exp(rng.uniform(-30, 30, (3, 4, 200)))
    w = rng.uniform(0, 1, 200)
    hi, lo = X._dd_weighted_sum(F, w)
    mpmath.mp.dps = 60
    for a in range(3):
        for b in range(4):
            terms = [mpmath.mpf(float(w[k])) * mpmath.mpf(float(F[a, b, k])) for k in range(200)]
            ex = mpmath.fsum(terms)
            bound = mpmath.fsum([abs(t) for t in terms]) * mpmath.mpf(2) ** -98  # ~ n * 2^-106
            assert abs((mpmath.mpf(float(hi[a, b])) + mpmath.mpf(float(lo[a, b]))) - ex) <= bound


def test_xform_d8_reproduces_paper_value():
    """End to end (cross + quadrature) on the paper's own setup: D_8 with 33-point
    Gauss-Legendre (§5.2) against the value printed in PAPER.md Fig. 5
    (tests/golden/paper_values.json, 32 digits): rank 24 gives ~1e-11."""
    import json
    import os
    from workloads import X_WORKLOADS
    wl = X_WORKLOADS["Dx8"]
    u, w = wl.grid()
    prob = X.Problem(wl.family, u, w, wl.rank_cap, wl.tol, wl.n_samples, wl.rook_iters, wl.seed)
    st, val, _ = X.run(prob, wl.sweeps)
    ref = float(json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))["D"]["8"])
    assert abs(val - ref) < 1e-9 * ref, (val, ref)


def test_folded_weights_integrate_to_the_same_grid_sum():
    """B = w x ... x w * f contracted with unit weights equals f contracted with w, both
    against the full Gauss-Legendre grid sum (small exact-enough cross)."""
    from workloads import FAMILY_DX, xform_grid
    x, w = xform_grid(4, 7)
    ref = ig.brute_force(FAMILY_DX, x, w)
    for fold in (False, True):
        prob = X.Problem(FAMILY_DX, x, w, 7, 1e-14, 64, 4, 3, fold)   # rank 7 = full rank here
        st, val, _ = X.run(prob, 8)
        assert abs(val - ref) < 1e-12 * abs(ref), (fold, val, ref)
