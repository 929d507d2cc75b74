"""Pins of oracle/cross.py against things other than itself (CPU only).

What fixes each expectation: the published splitmix64 test vector; an explicit list-based
Fisher-Yates; nestedness (eq. (4)); numpy.linalg inverses / determinants and
explicit Schur complements (independent arithmetic) for the cross and Alg. 1; exhaustive
swap search for maxvol local optimality; Theorem 1 (interpolation on nested crosses) and
Theorem 2 (exact recovery of exact-rank tensors); the TT formula eq. (3) evaluated entry by
entry against the full-grid sum for the §4.1 contraction.
"""
import itertools

import numpy as np
import pytest

from oracle import cross as X
from oracle import integrand as ig
from workloads import FAMILY_C, FAMILY_D, ising_grid


def make_problem(fam, d, n, L, cap, tol=1e-12, p=4, seed=7, delta=1e-2):
    u, w = ising_grid(d, n, L)
    return X.Problem(fam, u, w, cap, tol, p, delta, 0, seed)


# ---------------------------------------------------------------- counter-based RNG
def test_splitmix64_reference_vector():
    # splitmix64 from state 0 (Steele, Lea, Flood 2014; the JDK SplittableRandom mixer):
    # first outputs are the published test vector below.
    ref = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F, 0xF88BB8A8724C81EC]
    assert [X.splitmix64(0, c) for c in range(4)] == ref


def test_partial_fisher_yates_matches_explicit_shuffle():
    for M, r in [(10, 10), (257, 16), (4112, 16), (5, 1)]:
        got = X.partial_fisher_yates(99, 0, 5, 2, M, r)
        arr = list(range(M))
        for s in range(r):
            j = s + X.splitmix64(99, X.draw_ctr(0, 5, 2, s)) % (M - s)
            arr[s], arr[j] = arr[j], arr[s]
        assert got == arr[:r]
        assert len(set(got)) == r


# ---------------------------------------------------------------- initial pivots
@pytest.mark.parametrize("d,n,cap", [(2, 5, 8), (4, 9, 8), (5, 7, 16), (6, 3, 4)])
def test_initial_state_nested_distinct(d, n, cap):
    prob = make_problem(FAMILY_C, d, n, 4.0, cap)
    st = X.initial_state(prob)
    assert st.ranks == [min(cap, n ** (i + 1), n ** (d - 1 - i)) for i in range(d - 1)]
    for i, P in enumerate(st.piv):
        lefts = {tuple(r[:i + 1]) for r in P}
        rights = {tuple(r[i + 1:]) for r in P}
        assert len(lefts) == len(P) == len(rights)
        assert np.all((P >= 0) & (P < n))
        if i > 0:  # I_{<=i} subset of I_{<=i-1} x [n]   (eq. (4))
            prev = {tuple(r[:i]) for r in st.piv[i - 1]}
            assert all(t[:i] in prev for t in lefts)
        if i < d - 2:  # I_{>i} subset of [n] x I_{>i+1}
            nxt = {tuple(r[i + 2:]) for r in st.piv[i + 1]}
            assert all(t[1:] in nxt for t in rights)


# ---------------------------------------------------------------- fibers
def test_fiber_indexing_against_explicit_loop():
    prob = make_problem(FAMILY_D, 5, 7, 3.0, 4)
    st = X.initial_state(prob)
    for m in range(5):
        Lt = st.piv[m - 1] if m > 0 else None
        Rt = st.piv[m] if m < 4 else None
        F = X.fiber(prob, Lt, m, Rt)
        rx = 1 if Lt is None else len(Lt)
        ry = 1 if Rt is None else len(Rt)
        assert F.shape == (rx, ry, 7)
        for al in range(rx):
            for be in range(ry):
                for a in range(7):
                    t = (list(Lt[al][:m]) if m > 0 else []) + [a] + (list(Rt[be][m + 1:]) if m < 4 else [])
                    assert F[al, be, a] == ig.entries(FAMILY_D, prob.u, np.array([t]))[0]
        Mlr = X.fiber_matrix(F, X.DIR_LR)
        Mrl = X.fiber_matrix(F, X.DIR_RL)
        assert Mlr[2 * 7 + 3 if rx > 2 else 3, 0] == F[2 if rx > 2 else 0, 0, 3]
        assert Mrl[(ry - 1) * 7 + 5, rx - 1] == F[rx - 1, ry - 1, 5]


# ---------------------------------------------------------------- rank-revealing cross
def test_rrcross_exact_rank_and_B():
    rng = np.random.default_rng(0)
    for (m, c, k) in [(40, 10, 3), (100, 20, 7), (12, 12, 12)]:
        F = rng.standard_normal((m, k)) @ rng.standard_normal((k, c))
        I, J, B = X.rrcross(F, 1e-10, 64)
        assert len(I) == k and len(set(I)) == k and len(set(J)) == k
        Bref = F[:, J] @ np.linalg.inv(F[np.ix_(I, J)])
        assert np.max(np.abs(B - Bref)) < 1e-9 * max(1, np.max(np.abs(Bref)))
        assert np.array_equal(B[I, :], np.eye(k))  # exact identity on the pivot rows
        # cap is honoured
        I2, J2, _ = X.rrcross(F, 1e-10, 2)
        assert len(I2) == 2 and I2 == I[:2] and J2 == J[:2]
    I, J, B = X.rrcross(np.zeros((5, 3)), 1e-12, 4)
    assert I == [] and J == []


def test_rrcross_is_complete_pivoting():
    """Pivot s+1 is the max |Schur complement| entry after pivots 1..s (explicit formula)."""
    rng = np.random.default_rng(1)
    F = rng.standard_normal((30, 8)) * np.exp(rng.standard_normal((30, 1)))
    I, J, _ = X.rrcross(F, 1e-14, 8)
    for s in range(len(I)):
        if s == 0:
            Rs = F
        else:
            Is, Js = I[:s], J[:s]
            Rs = F - F[:, Js] @ np.linalg.solve(F[np.ix_(Is, Js)], F[Is, :])
            Rs[Is, :] = 0
            Rs[:, Js] = 0
        assert abs(Rs[I[s], J[s]]) >= np.max(np.abs(Rs)) * (1 - 1e-9)


# ---------------------------------------------------------------- maxvol (Alg. 1)
def test_maxvol_paper_toy_example():
    # A = [[1],[3]], J = {0}, I = {0}: B = [1; 3] -> swap to I = {1}, volume x3
    F = np.array([[1.0], [3.0]])
    B = F / F[0, 0]
    I, B2, nsw = X.maxvol(B, [0], 1e-2, 10)
    assert I == [1] and nsw == 1
    assert np.allclose(B2, F / F[1, 0])


def test_maxvol_volume_growth_and_bound():
    rng = np.random.default_rng(2)
    for trial in range(20):
        m, r = rng.integers(8, 60), rng.integers(1, 7)
        F = rng.standard_normal((m, r))
        I0 = list(rng.choice(m, r, replace=False))
        if abs(np.linalg.det(F[I0])) < 1e-6:
            continue
        B0 = F @ np.linalg.inv(F[I0])
        I = list(I0)
        vol = abs(np.linalg.det(F[I]))
        for step in range(1, 200):
            Inew, Bnew, nsw = X.maxvol(B0, I0, 1e-2, step)
            if nsw < step:  # converged
                Bref = F @ np.linalg.inv(F[Inew])
                assert np.max(np.abs(Bref)) <= 1 + 1e-2 + 1e-9
                assert np.max(np.abs(Bnew - Bref)) < 1e-9
                break
            v = abs(np.linalg.det(F[Inew]))
            assert v > vol * (1 + 1e-2) * (1 - 1e-9)  # every swap grows the volume (Alg. 1)
            vol = v


def test_maxvol_local_optimality_exhaustive():
    rng = np.random.default_rng(3)
    for trial in range(30):
        m, r = 9, 2
        F = rng.standard_normal((m, r))
        I, J, B = X.rrcross(F, 1e-14, r)
        I, B, nsw = X.maxvol(B, I, 1e-2, 100)
        v = abs(np.linalg.det(F[I]))
        for j in range(r):
            for i in range(m):
                if i in I:
                    continue
                I2 = list(I)
                I2[j] = i
                assert abs(np.linalg.det(F[I2])) <= v * (1 + 1e-2) * (1 + 1e-12)


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


def test_interpolation_theorem1_on_nested_init():
    """Theorem 1: nested crosses interpolate their fibers."""
    u, w = ising_grid(4, 6, 3.0)
    prob = AsymProblem(FAMILY_C, u, w, 3, 1e-12, 4, 1e-2, 0, 7)
    st = X.initial_state(prob)  # nested by construction
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
    prob = ExactRankProblem(FAMILY_C, u, w, 4, 1e-13, 4, 1e-2, 0, 5)
    st = X.initial_state(prob)
    st = X.sweep(prob, st)
    assert max(st.ranks) <= 2  # truncation finds the exact rank
    val, *_ = X.integrate(prob, st)
    d, n = 4, 7
    tot = 0.0
    for idx in itertools.product(range(n), repeat=d):
        wt = np.prod([w[j][idx[j]] for j in range(d)])
        tot += wt * prob.A(np.array([idx]))[0]
    assert abs(val - tot * ig.prefactor(d)) <= 1e-12 * abs(val)


def test_half_sweep_invariants():
    prob = make_problem(FAMILY_D, 5, 17, 6.0, 6, tol=1e-11, p=3)
    st = X.initial_state(prob)
    for s in range(2):
        for direction in (X.DIR_LR, X.DIR_RL):
            new = X.half_sweep(prob, st, direction)
            for i, P in enumerate(new.piv):
                assert 1 <= len(P) <= prob.rank_cap
                assert len({tuple(r[:i + 1]) for r in P}) == len(P)
                assert len({tuple(r[i + 1:]) for r in P}) == len(P)
                M = X.intersection(prob, new, i)
                assert abs(np.linalg.det(M)) > 0
                if direction == X.DIR_LR and i > 0:
                    # new left parts come from the OLD I_{<=i-1} x [n]   (§3.4 relaxation)
                    old = {tuple(r[:i]) for r in st.piv[i - 1]}
                    assert all(tuple(r[:i]) in old for r in P)
                if direction == X.DIR_RL and i < prob.d - 2:
                    old = {tuple(r[i + 2:]) for r in st.piv[i + 1]}
                    assert all(tuple(r[i + 2:]) in old for r in P)
            st = new
        st.sweep += 1


def test_parallel_partition_equals_all_at_once():
    """Alg. 6: updating disjoint interface chunks separately and merging equals one
    half-sweep over all interfaces (each interface only reads the previous state)."""
    prob = make_problem(FAMILY_C, 7, 9, 4.0, 5)
    st = X.initial_state(prob)
    full = X.half_sweep(prob, st, X.DIR_LR)
    merged = st.copy()
    for chunk in ([0, 1], [2, 3, 4], [5]):
        part = X.half_sweep(prob, st, X.DIR_LR, chunk)
        for i in chunk:
            merged.piv[i] = part.piv[i]
    for a, b in zip(full.piv, merged.piv):
        assert np.array_equal(a, b)


def test_c4_converges_toward_brute_force():
    """Sanity of the whole pipeline: C_4 at rank cap 16 approaches the full-grid sum."""
    prob = make_problem(FAMILY_C, 4, 33, 8.0, 16, tol=1e-13)
    st, val, _ = X.run(prob, 4)
    ref = ig.brute_force(FAMILY_C, prob.u, prob.w)
    assert abs(val - ref) < 1e-6 * ref


def test_integrate_exact_agrees_with_fp64_when_well_conditioned():
    """R9: the near-exact contraction equals the fp64 one to rounding on a well-conditioned
    cross, and equals the full-grid sum of the TT reconstruction (eq. (3))."""
    prob = make_problem(FAMILY_D, 3, 6, 3.0, 4)
    st = X.sweep(prob, X.initial_state(prob))
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
