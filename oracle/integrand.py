"""ORACLE (test infrastructure only): the Ising integrands as tensor entries.

Definitions (readings R1-R3):

* BASELINE.json configs state the integrals in the Bailey-Borwein-Crandall t-form
      C_d = (4/d!) int_{R^d} dt / (sum_j 2cosh t_j)^2
      D_d = (4/d!) int_{R^d} prod_{i<j} tanh^2((t_i-t_j)/2) dt / (sum_j 2cosh t_j)^2
  with "u = e^t substitution".  With u_j = e^{t_j}:  2cosh t_j = u_j + 1/u_j and
  tanh((t_i-t_j)/2) = (u_i-u_j)/(u_i+u_j).  These are the same integrals as PAPER.md
  §5.1 eq. (9)-(10) (lines 843-851; the paper's x-variables are ratios of consecutive
  u's, cf. its A_d with factors (1-x_{i+1}..x_j)/(1+x_{i+1}..x_j) = (u_i-u_j)/(u_i+u_j)).
  tests/test_oracle_integrand.py pins the two forms against each other.

* The tensor whose TT cross is built is the raw integrand on the grid (no weights folded,
  PAPER.md §4.1; the folded variant of lines 701-706 is offered for the
  x-form families only, oracle.cross.Problem(fold=True), R2):
      A(i_1..i_d) = f(u_{1,i_1}, ..., u_{d,i_d}),   f = P / S^2,
      S = sum_j (u_j + 1/u_j),      P = prod_{i<j} rho(u_i, u_j)  (P = 1 for family C),
      rho(x, y) = q*q,  q = (max(x,y) - min(x,y)) / (max(x,y) + min(x,y)).
  The prefactor 4/d! multiplies the integral only.

* Floating point (reading R3): every entry is *the same fp64 number* however the
  coordinates are ordered:  S is the correctly rounded exact sum of the per-node
  c_j = fl(u_j + fl(1/u_j));  P is the correctly rounded exact product of the per-pair
  rho (computed here in double-double with an exact power-of-two exponent, error
  <= N_pairs * 2^-100 relative before the single final rounding);  then
  f = fl(P / fl(S*S)).  Making the entry a function of the multiset of coordinates
  (not of the evaluation order) is what lets the CUDA path factorize the product over a
  fiber's frozen coordinates and still reproduce these bits, so that pivot decisions can
  be compared bit-exactly.
"""
from __future__ import annotations

import math

import numpy as np

FAMILY_C = 0
FAMILY_D = 1
FAMILY_CX = 2
FAMILY_DX = 3
FAMILY_EX = 4
X_FAMILIES = (FAMILY_CX, FAMILY_DX, FAMILY_EX)

_TWO52 = float(2 ** 52)
_SPLIT = 134217729.0  # 2^27 + 1, Veltkamp/Dekker splitter
_RESCALE_EXP = 500
_RESCALE_THR = 2.0 ** -_RESCALE_EXP


# --------------------------------------------------------------------------------------
# per-node quantities
# --------------------------------------------------------------------------------------
def node_c(u):
    """c = fl(u + fl(1/u)) = 2cosh(t) on the u-node (BASELINE.json 'u=e^t substitution')."""
    u = np.asarray(u, dtype=np.float64)
    return u + 1.0 / u


def rho(x, y):
    """rho(x,y) = q*q, q = (hi-lo)/(hi+lo); equals tanh^2((t_x-t_y)/2) for x=e^{t_x}."""
    hi = np.maximum(x, y)
    lo = np.minimum(x, y)
    q = (hi - lo) / (hi + lo)
    return q * q


# --------------------------------------------------------------------------------------
# exact sum of c-values (correctly rounded), vectorised over entries
# --------------------------------------------------------------------------------------
def exact_sum_rn(cvals):
    """Correctly rounded sum of the last axis of ``cvals`` (all entries must be >= 1).

    Each c >= 1 has ulp(c) >= 2^-52, so c = H + Lo*2^-52 with integers H = floor(c) and
    Lo = (c - H)*2^52 < 2^52, both exact.  Integer sums are exact; one carry normalisation
    and one fp addition of two exactly representable doubles give the single rounding.
    """
    c = np.asarray(cvals, dtype=np.float64)
    if c.size and not np.all(c >= 1.0):
        raise ValueError("exact_sum_rn requires all terms >= 1")
    H = np.floor(c)
    Lo = ((c - H) * _TWO52).astype(np.int64)
    Hs = H.astype(np.int64).sum(axis=-1)
    Ls = Lo.sum(axis=-1)
    Hs = Hs + (Ls >> 52)
    Ls = Ls & ((1 << 52) - 1)
    return Hs.astype(np.float64) + Ls.astype(np.float64) * (1.0 / _TWO52)


# --------------------------------------------------------------------------------------
# double-double product with exact binary exponent
# --------------------------------------------------------------------------------------
def _split(a):
    c = _SPLIT * a
    hi = c - (c - a)
    return hi, a - hi


def _two_prod(a, b):
    p = a * b
    ah, al = _split(a)
    bh, bl = _split(b)
    err = ((ah * bh - p) + ah * bl + al * bh) + al * bl
    return p, err


class DDProduct:
    """Running product hi+lo (double-double) times 2^e, for factors in [0, 1]."""

    def __init__(self, shape):
        self.hi = np.ones(shape, dtype=np.float64)
        self.lo = np.zeros(shape, dtype=np.float64)
        self.e = np.zeros(shape, dtype=np.int64)

    def mul(self, b):
        b = np.broadcast_to(np.asarray(b, dtype=np.float64), self.hi.shape)
        p, err = _two_prod(self.hi, b)
        t = self.lo * b + err
        hi = p + t
        lo = t - (hi - p)
        small = (hi < _RESCALE_THR) & (hi != 0.0)
        if np.any(small):
            hi = np.where(small, hi * 2.0 ** _RESCALE_EXP, hi)
            lo = np.where(small, lo * 2.0 ** _RESCALE_EXP, lo)
            self.e = self.e - np.where(small, _RESCALE_EXP, 0)
        self.hi, self.lo = hi, lo

    def rounded(self):
        """fl(exact product): round hi+lo once, then apply the exact exponent."""
        return np.ldexp(self.hi + self.lo, self.e)


# --------------------------------------------------------------------------------------
# the tensor entry A(i) and brute force
# --------------------------------------------------------------------------------------
def entries(family, u_nodes, idx):
    """A(idx) for integer multi-indices ``idx`` of shape (..., d); u_nodes has shape (d, n).

    Plain evaluation of the definition: S over all d coordinates, P over all d(d-1)/2
    pairs in lexicographic order (the order does not matter for the rounded result).
    """
    if family in X_FAMILIES:
        return entries_x(family, u_nodes, idx)
    u_nodes = np.asarray(u_nodes, dtype=np.float64)
    idx = np.asarray(idx)
    d = idx.shape[-1]
    U = np.stack([u_nodes[j][idx[..., j]] for j in range(d)], axis=-1) if d else np.zeros(idx.shape)
    S = exact_sum_rn(node_c(U))
    SS = S * S
    if family == FAMILY_C:
        return 1.0 / SS
    if family != FAMILY_D:
        raise ValueError(f"unknown family {family}")
    prod = DDProduct(idx.shape[:-1])
    for i in range(d):
        for j in range(i + 1, d):
            prod.mul(rho(U[..., i], U[..., j]))
    return prod.rounded() / SS


def entries_x(family, x_nodes, idx):
    """The paper's x-form integrands (eq. (9)-(11), lines 843-851) at the grid
    multi-indices ``idx`` (..., m), m = d-1 modes holding x_2..x_d:

        B_d = (1 + sum_{k=2}^d x_2..x_k)^{-1} (1 + sum_{k=2}^d x_k..x_d)^{-1}
        A_d = prod_{1<=i<j<=d} ((1 - x_{i+1}..x_j) / (1 + x_{i+1}..x_j))^2
        C: B_d,  D: A_d * B_d,  E: A_d.

    Plain fp64 in this fixed operation order (the CUDA path repeats it; no fused
    multiply-add): S1 accumulates the prefix products left to right, S2 the suffix
    products right to left, B = 1 / (S1 * S2); A multiplies q*q, q = (1-p)/(1+p), over
    i = 1..d-1 then j = i+1..d with the running product p = x_{i+1}..x_j.
    """
    x_nodes = np.asarray(x_nodes, dtype=np.float64)
    idx = np.asarray(idx)
    m = idx.shape[-1]
    X = [x_nodes[j][idx[..., j]] for j in range(m)]
    shape = idx.shape[:-1]
    A = np.ones(shape)
    if family in (FAMILY_DX, FAMILY_EX):
        for i in range(m):           # paper i' = i + 1 (x_{i'+1} = X[i])
            p = np.ones(shape)
            for j in range(i, m):    # paper j' = j + 2, p = x_{i'+1}..x_{j'}
                p = p * X[j]
                q = (1.0 - p) / (1.0 + p)
                A = A * (q * q)
    if family == FAMILY_EX:
        return A
    S1 = np.ones(shape)
    p = np.ones(shape)
    for k in range(m):
        p = p * X[k]
        S1 = S1 + p
    S2 = np.ones(shape)
    p = np.ones(shape)
    for k in range(m - 1, -1, -1):
        p = p * X[k]
        S2 = S2 + p
    B = 1.0 / (S1 * S2)
    if family == FAMILY_CX:
        return B
    if family != FAMILY_DX:
        raise ValueError(f"unknown family {family}")
    return A * B


def prefactor(d, family=FAMILY_C):
    """Integral prefactor: 4/d! of the (4/d!)-normalised t-form (BASELINE.json configs), 2
    for the x-form (eq. (9)-(11)).  For the x-form `d` is the number of modes."""
    if family in X_FAMILIES:
        return 2.0
    return 4.0 / math.factorial(d)


def brute_force(family, u_nodes, weights, chunk=1 << 21):
    """Full tensor-product quadrature sum (§4.1 eq. (5)) times 4/d!.

    Exponential in d: only for d <= 4 with moderate n.
    """
    u_nodes = np.asarray(u_nodes, dtype=np.float64)
    weights = np.asarray(weights, dtype=np.float64)
    d, n = u_nodes.shape
    total = n ** d
    acc = 0.0
    for start in range(0, total, chunk):
        flat = np.arange(start, min(total, start + chunk), dtype=np.int64)
        idx = np.empty((flat.size, d), dtype=np.int64)
        rem = flat.copy()
        for j in range(d - 1, -1, -1):
            idx[:, j] = rem % n
            rem //= n
        w = np.ones(flat.size)
        for j in range(d):
            w = w * weights[j][idx[:, j]]
        acc += float(np.sum(w * entries(family, u_nodes, idx)))
    return acc * prefactor(d, family)
