"""Seeded synthetic input generators shared by the CUDA path, the oracle tests and bench.py.

This module holds NONE of the method's arithmetic (no integrand, no cross, no maxvol,
no contraction).  It only builds the *problem statement* the paper's method takes
(§4.1 "Tensor product quadratures", lines 666-672): a tensor-product grid of
nodes and quadrature weights, plus the workload table of BASELINE.json.

Grid recipe (BASELINE.json ``configs``): the Ising integrals are taken in the
Bailey-Borwein-Crandall form  C_d = (4/d!) int_{R^d} dt / (sum_j 2cosh t_j)^2  with the
substitution u = e^t, i.e. the integrand is evaluated on u-nodes.  The 1-D rule is the
composite trapezoid on t in [-L, L] with n points:
    h = 2L/(n-1),  t_a = -L + a*h,  w_a = h (w_0 = w_{n-1} = h/2),  u_a = exp(t_a).
For the configured (L, n) pairs h is a dyadic rational, so t_a is exact and the grid is
exactly symmetric.  exp() is evaluated once here, on the host, so that the oracle and the
CUDA path consume bit-identical u-nodes (the nodes are an input, like a dataset).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

FAMILY_C = 0  # C_d : f = 1/(sum_j (u_j + 1/u_j))^2                         (t-form, u-nodes)
FAMILY_D = 1  # D_d : f = prod_{i<j} ((u_i-u_j)/(u_i+u_j))^2 / (sum_j (u_j + 1/u_j))^2
# the paper's own x-form (eq. (9)-(11)) on [0,1]^{d-1}: the tensor has d-1 modes
# (x_2..x_d) and the integral prefactor is 2
FAMILY_CX = 2  # C_d = 2 int B_d
FAMILY_DX = 3  # D_d = 2 int A_d B_d
FAMILY_EX = 4  # E_d = 2 int A_d
FAMILY_NAMES = {FAMILY_C: "C", FAMILY_D: "D", FAMILY_CX: "Cx", FAMILY_DX: "Dx", FAMILY_EX: "Ex"}
X_FAMILIES = (FAMILY_CX, FAMILY_DX, FAMILY_EX)


def trapezoid_t_grid(n: int, L: float):
    """Composite trapezoid rule on [-L, L] with n >= 2 points: (t, w)."""
    if n < 2:
        raise ValueError("trapezoid grid needs n >= 2")
    h = 2.0 * L / (n - 1)
    t = -L + h * np.arange(n, dtype=np.float64)
    w = np.full(n, h, dtype=np.float64)
    w[0] = w[-1] = h / 2
    return t, w


def gauss_legendre01(n: int):
    """n-point Gauss-Legendre rule on [0, 1] (nodes ascending, weights summing to 1);
    PAPER.md §5.2 "tensor product of one-dimensional Gauss--Legendre quadratures"."""
    x, w = np.polynomial.legendre.leggauss(n)
    return (x + 1.0) / 2.0, w / 2.0


def xform_grid(d: int, n: int):
    """x-nodes (d-1, n) and weights (d-1, n) of the x-form integrals (eq. (9)-(11)):
    one Gauss-Legendre rule per variable x_2..x_d."""
    x, w = gauss_legendre01(n)
    return np.ascontiguousarray(np.tile(x, (d - 1, 1))), np.ascontiguousarray(np.tile(w, (d - 1, 1)))


def ising_grid(d: int, n: int, L: float):
    """u-nodes (d, n) and weights (d, n) for a d-mode Ising problem (same rule per mode)."""
    t, w = trapezoid_t_grid(n, L)
    u = np.exp(t)
    return np.ascontiguousarray(np.tile(u, (d, 1))), np.ascontiguousarray(np.tile(w, (d, 1)))


@dataclass(frozen=True)
class Workload:
    name: str
    family: int
    d: int
    n: int
    L: float
    rank_cap: int
    tol: float
    sweeps: int
    n_samples: int = 32      # |L| of Alg. 2 line 1 (R6)
    rook_iters: int = 4      # rook rounds of Alg. 2 (R6)
    seed: int = 20190327
    note: str = ""
    fold: bool = False       # cross on w x ... x w * f (§4.1)

    @property
    def alg6_sweeps(self) -> int:
        """Dimension-parallel sweeps of PAPER.md Alg. 6 run by one solve.  Each adds at most one
        pivot per superblock, so one BASELINE 'sweep' is ceil((cap-1)/sweeps) Alg. 6 sweeps:
        enough to reach the rank cap from rank 1 in the configured number (R7)."""
        return self.sweeps * max(1, -(-(self.rank_cap - 1) // self.sweeps))

    @property
    def modes(self) -> int:
        """Modes of the tensor: d for the t-form, d-1 (x_2..x_d) for the x-form."""
        return self.d - 1 if self.family in X_FAMILIES else self.d

    def grid(self):
        if self.family in X_FAMILIES:
            return xform_grid(self.d, self.n)
        return ising_grid(self.d, self.n, self.L)

    def prefactor(self) -> float:
        return 2.0 if self.family in X_FAMILIES else 4.0 / math.factorial(self.d)


# BASELINE.json configs[0..4].  `sweeps` is the BASELINE sweep count (4 where a config
# states none, R7); `alg6_sweeps` the dimension-parallel sweeps it stands for.
WORKLOADS = {
    "C4": Workload("C4", FAMILY_C, 4, 129, 20.0, 8, 1e-10, 4,
                   note="configs[0]: C_4, 129-pt trapezoid on [-20,20], rank cap 8, tol 1e-10"),
    "D5": Workload("D5", FAMILY_D, 5, 257, 20.0, 16, 1e-11, 4,
                   note="configs[1]: D_5, 257-pt trapezoid on [-20,20], rank cap 16, tol 1e-11"),
    "C10": Workload("C10", FAMILY_C, 10, 257, 20.0, 32, 1e-12, 4,
                    note="configs[2]: C_10, 257-pt trapezoid on [-20,20], rank cap 32, tol 1e-12, 4 sweeps"),
    "D20": Workload("D20", FAMILY_D, 20, 513, 24.0, 64, 1e-12, 4,
                    note="configs[3]: D_20, 513-pt trapezoid on [-24,24], rank cap 64, tol 1e-12"),
    "C200": Workload("C200", FAMILY_C, 200, 257, 20.0, 32, 1e-12, 6,
                     note="configs[4]: C_200, 257-pt trapezoid on [-20,20], rank cap 32, 6 sweeps"),
}

# The paper's own setup (§5.2-5.4): x-form integrands, n-point Gauss-Legendre per
# variable.  Not BASELINE configs -- validation workloads for the "next" row of DESIGN.md §8
# (D_8 is printed in PAPER.md Fig. 5 to 32 digits; C_d -> 2 exp(-2 gamma)).
X_WORKLOADS = {
    "Dx8": Workload("Dx8", FAMILY_DX, 8, 33, 0.0, 24, 1e-14, 24, note="D_8, 33-pt Gauss-Legendre, rank cap 24"),
    "Cx64": Workload("Cx64", FAMILY_CX, 64, 33, 0.0, 16, 1e-14, 16, note="C_64, 33-pt Gauss-Legendre, rank cap 16"),
    "Ex6": Workload("Ex6", FAMILY_EX, 6, 33, 0.0, 20, 1e-14, 20, note="E_6, 33-pt Gauss-Legendre, rank cap 20"),
    "Dx8f": Workload("Dx8f", FAMILY_DX, 8, 33, 0.0, 24, 1e-14, 24, fold=True,
                     note="D_8, 33-pt Gauss-Legendre, rank cap 24, weights folded into the tensor"),
}
