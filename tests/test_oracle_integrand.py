"""Pins of oracle/integrand.py against things other than itself (CPU only).

Each test names what fixes the expected value: libm transcendental identities, Python's
correctly-rounded math.fsum, mpmath exact products, closed forms (tests/golden), the
paper's own x-form (eq. (9)-(10)), and the paper's printed D_d values.
"""
import json
import math
import os

import mpmath
import numpy as np
import pytest

from oracle import integrand as ig
from workloads import FAMILY_C, FAMILY_D, ising_grid, trapezoid_t_grid

GOLD = os.path.join(os.path.dirname(__file__), "golden")
mpmath.mp.dps = 40


def L_m3_2():
    # Dirichlet L-function of the non-principal character mod 3 at s=2
    return (mpmath.zeta(2, mpmath.mpf(1) / 3) - mpmath.zeta(2, mpmath.mpf(2) / 3)) / 9


CLOSED = {
    ("C", 1): lambda: mpmath.mpf(2),
    ("C", 2): lambda: mpmath.mpf(1),
    ("C", 3): L_m3_2,
    ("C", 4): lambda: 7 * mpmath.zeta(3) / 12,
    ("D", 2): lambda: mpmath.mpf(1) / 3,
    ("D", 3): lambda: 8 + 4 * mpmath.pi ** 2 / 3 - 27 * L_m3_2(),
    ("D", 4): lambda: 4 * mpmath.pi ** 2 / 9 - mpmath.mpf(1) / 6 - 7 * mpmath.zeta(3) / 2,
}


def test_node_c_is_2cosh():
    t, _ = trapezoid_t_grid(257, 20.0)
    c = ig.node_c(np.exp(t))
    ref = np.array([2 * math.cosh(x) for x in t])
    assert np.max(np.abs(c - ref) / ref) < 4e-16


def test_rho_is_tanh_squared():
    t, _ = trapezoid_t_grid(129, 20.0)
    u = np.exp(t)
    rng = np.random.default_rng(0)
    a, b = rng.integers(0, 129, 2000), rng.integers(0, 129, 2000)
    got = ig.rho(u[a], u[b])
    ref = np.array([math.tanh((t[x] - t[y]) / 2) ** 2 for x, y in zip(a, b)])
    nz = ref > 1e-3
    assert np.all(got[~nz] <= 1e-3 * 1.01)
    assert np.max(np.abs(got[nz] - ref[nz]) / ref[nz]) < 1e-13
    assert np.all(got[a == b] == 0.0)
    assert np.array_equal(ig.rho(u[a], u[b]), ig.rho(u[b], u[a]))  # symmetric bitwise


def test_exact_sum_is_correctly_rounded_and_order_free():
    rng = np.random.default_rng(1)
    for d in (1, 2, 5, 20, 200):
        c = ig.node_c(np.exp(rng.uniform(-24, 24, size=(300, d))))
        got = ig.exact_sum_rn(c)
        ref = np.array([math.fsum(row) for row in c])  # Shewchuk: correctly rounded
        assert np.array_equal(got, ref)
        perm = rng.permutation(d)
        assert np.array_equal(ig.exact_sum_rn(c[:, perm]), got)


def test_dd_product_is_correctly_rounded():
    rng = np.random.default_rng(2)
    for npairs in (1, 3, 10, 190, 1200):
        vals = rng.uniform(0.0, 1.0, size=(40, npairs)) ** 3
        vals[0, :] = 0.5  # exact power of two
        if npairs >= 190:
            vals[1, :] = 1e-3  # underflows fp64 without the exponent bookkeeping
        p = ig.DDProduct((40,))
        for j in range(npairs):
            p.mul(vals[:, j])
        got = p.rounded()
        for r in range(40):
            exact = mpmath.fprod([mpmath.mpf(float(x)) for x in vals[r]])
            assert got[r] == float(exact), (npairs, r)


def test_entries_are_symmetric_functions_bitwise():
    u, _ = ising_grid(7, 65, 16.0)
    rng = np.random.default_rng(3)
    idx = rng.integers(0, 65, size=(500, 7))
    for fam in (FAMILY_C, FAMILY_D):
        base = ig.entries(fam, u, idx)
        for _ in range(3):
            perm = rng.permutation(7)
            assert np.array_equal(ig.entries(fam, u, idx[:, perm]), base)


def test_entries_direct_formula_small():
    # d=2, by hand: C: 1/(c1+c2)^2 ; D: rho(u1,u2)/(c1+c2)^2 ; t-form identities
    t1, t2 = 0.375, -1.25
    u = np.array([[math.exp(t1)], [math.exp(t2)]])
    idx = np.array([[0, 0]])
    S = 2 * math.cosh(t1) + 2 * math.cosh(t2)
    assert abs(ig.entries(FAMILY_C, u, idx)[0] * S * S - 1) < 1e-15
    dref = math.tanh((t1 - t2) / 2) ** 2 / S ** 2
    assert abs(ig.entries(FAMILY_D, u, idx)[0] / dref - 1) < 1e-14
    # D vanishes whenever two coordinates coincide
    u3, _ = ising_grid(4, 9, 4.0)
    assert ig.entries(FAMILY_D, u3, np.array([[1, 5, 1, 7]]))[0] == 0.0


@pytest.mark.parametrize("fam,d,n,L,tol", [
    # tolerances ~5x the observed trapezoid error of each grid (exponential in 1/h)
    ("C", 1, 129, 20.0, 1e-11),
    ("C", 2, 129, 20.0, 1e-14),
    ("C", 3, 129, 20.0, 1e-13),
    ("C", 4, 65, 14.0, 1e-7),
    ("D", 2, 129, 20.0, 1e-14),
    ("D", 3, 129, 20.0, 1e-12),
    ("D", 4, 65, 14.0, 2e-6),
])
def test_brute_force_matches_closed_forms(fam, d, n, L, tol):
    """Full-grid trapezoid sums of the oracle integrand against the closed forms."""
    u, w = ising_grid(d, n, L)
    fid = FAMILY_C if fam == "C" else FAMILY_D
    got = ig.brute_force(fid, u, w)
    ref = float(CLOSED[(fam, d)]())
    assert abs(got - ref) <= tol * abs(ref), (got, ref)


def _gauss_legendre01(n):
    x, w = np.polynomial.legendre.leggauss(n)
    return (x + 1) / 2, w / 2


def test_t_form_equals_paper_x_form():
    """Reading R1: the (4/d!) t-form on u=e^t equals PAPER.md eq. (9)/(10) (x-form).

    eq. (9):  C_d = 2 int_{[0,1]^{d-1}} B_d,  eq. (10): D_d = 2 int A_d B_d  with
    B_d = (1+sum_k x_2..x_k)^-1 (1+sum_k x_k..x_d)^-1 and
    A_d = prod_{i<j} ((1-x_{i+1}..x_j)/(1+x_{i+1}..x_j))^2  (lines 843-851).
    """
    xg, wg = _gauss_legendre01(60)
    for d in (2, 3):
        grids = np.meshgrid(*([xg] * (d - 1)), indexing="ij")
        X = {k + 2: g.ravel() for k, g in enumerate(grids)}  # x_2..x_d
        W = np.ones_like(X[2])
        for g in np.meshgrid(*([wg] * (d - 1)), indexing="ij"):
            W = W * g.ravel()

        def prod(a, b):
            out = np.ones_like(X[2])
            for k in range(a, b + 1):
                out = out * X[k]
            return out
        B = 1.0 / (1 + sum(prod(2, k) for k in range(2, d + 1)))
        B = B / (1 + sum(prod(k, d) for k in range(2, d + 1)))
        A = np.ones_like(B)
        for i in range(1, d + 1):
            for j in range(i + 1, d + 1):
                p = prod(i + 1, j)
                A = A * ((1 - p) / (1 + p)) ** 2
        c_x = 2 * float(np.sum(W * B))
        d_x = 2 * float(np.sum(W * A * B))
        u, w = ising_grid(d, 129, 20.0)
        assert abs(ig.brute_force(FAMILY_C, u, w) - c_x) < 1e-12 * c_x
        assert abs(ig.brute_force(FAMILY_D, u, w) - d_x) < 1e-11 * d_x


def test_paper_delta_consistency():
    """PAPER.md eq. (14): Delta = (D_128/D_256)^(1/128) from its own printed values."""
    vals = json.load(open(os.path.join(GOLD, "paper_values.json")))
    d128 = mpmath.mpf(vals["D"]["128"])
    d256 = mpmath.mpf(vals["D"]["256"])
    delta = (d128 / d256) ** (mpmath.mpf(1) / 128)
    assert abs(delta - mpmath.mpf(vals["Delta"])) < 1e-8


# ---------------------------------------------------------------- x-form (eq. (9)-(11))
def _xform_brute(fam, d, n):
    from workloads import xform_grid
    x, w = xform_grid(d, n)
    return ig.brute_force(fam, x, w)


@pytest.mark.parametrize("fam,d,n,tol", [("C", 2, 20, 1e-14), ("C", 3, 24, 1e-13), ("C", 4, 24, 1e-12),
                                         ("D", 2, 20, 1e-14), ("D", 3, 24, 1e-12), ("D", 4, 24, 1e-10)])
def test_xform_gauss_legendre_matches_closed_forms(fam, d, n, tol):
    """Full Gauss-Legendre tensor sums of the x-form oracle integrand (eq. (9)-(10))
    against the closed forms of BASELINE.json north_star (no reading involved)."""
    from workloads import FAMILY_CX, FAMILY_DX
    got = _xform_brute(FAMILY_CX if fam == "C" else FAMILY_DX, d, n)
    ref = float(CLOSED[(fam, d)]())
    assert abs(got - ref) <= tol * abs(ref), (got, ref)


def test_xform_e2_closed_form():
    """E_2 = 2 int_0^1 ((1-x)/(1+x))^2 dx = 6 - 8 log 2 (elementary antiderivative)."""
    from workloads import FAMILY_EX
    assert abs(_xform_brute(FAMILY_EX, 2, 20) - (6 - 8 * math.log(2))) < 1e-14


def test_xform_e3_numerical_quadrature():
    """E_3 = 2 int_{[0,1]^2} A_3 against mpmath's own adaptive quadrature."""
    from workloads import FAMILY_EX
    f = lambda x2, x3: ((1 - x2) / (1 + x2)) ** 2 * ((1 - x2 * x3) / (1 + x2 * x3)) ** 2 * ((1 - x3) / (1 + x3)) ** 2
    ref = 2 * mpmath.quad(f, [0, 1], [0, 1])
    assert abs(_xform_brute(FAMILY_EX, 3, 24) - float(ref)) < 1e-12 * float(ref)


def test_xform_entry_order_is_plain_fp64():
    """The x-form entry is exactly the documented operation sequence (retyped with Python
    floats, scalar by scalar)."""
    from workloads import FAMILY_CX, FAMILY_DX, xform_grid
    x, _ = xform_grid(5, 9)
    rng = np.random.default_rng(3)
    for _ in range(50):
        idx = rng.integers(0, 9, 4)
        X = [float(x[j][idx[j]]) for j in range(4)]
        S1, p = 1.0, 1.0
        for v in X:
            p = p * v
            S1 = S1 + p
        S2, p = 1.0, 1.0
        for v in reversed(X):
            p = p * v
            S2 = S2 + p
        B = 1.0 / (S1 * S2)
        A = 1.0
        for i in range(4):
            p = 1.0
            for j in range(i, 4):
                p = p * X[j]
                q = (1.0 - p) / (1.0 + p)
                A = A * (q * q)
        assert ig.entries(FAMILY_CX, x, idx[None])[0] == B
        assert ig.entries(FAMILY_DX, x, idx[None])[0] == A * B
