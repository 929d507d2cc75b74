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

FAMILY_C = 0  # C_d : f = 1/(sum_j (u_j + 1/u_j))^2
FAMILY_D = 1  # D_d : f = prod_{i<j} ((u_i-u_j)/(u_i+u_j))^2 / (sum_j (u_j + 1/u_j))^2
FAMILY_NAMES = {FAMILY_C: "C", FAMILY_D: "D"}


def trapezoid_t_grid(n: int, L: float):
    """Composite trapezoid rule on [-L, L] with n >= 2 points: (t, w)."""
    if n < 2:
        raise ValueError("trapezoid grid needs n >= 2")
    h = 2.0 * L / (n - 1)
    t = -L + h * np.arange(n, dtype=np.float64)
    w = np.full(n, h, dtype=np.float64)
    w[0] = w[-1] = h / 2
    return t, w


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

    @property
    def alg6_sweeps(self) -> int:
        """Dimension-parallel sweeps of PAPER.md Alg. 6 run by one solve.  Each adds at most one
        pivot per superblock, so one BASELINE 'sweep' is ceil((cap-1)/sweeps) Alg. 6 sweeps:
        enough to reach the rank cap from rank 1 in the configured number (R7)."""
        return self.sweeps * max(1, -(-(self.rank_cap - 1) // self.sweeps))

    def grid(self):
        return ising_grid(self.d, self.n, self.L)

    def prefactor(self) -> float:
        return 4.0 / math.factorial(self.d)


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
