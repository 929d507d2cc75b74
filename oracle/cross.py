"""ORACLE (test infrastructure only): dimension-parallel greedy TT cross + TT quadrature.

Follows DESIGN.md §2 step by step.  Notation: modes m = 0..d-1 (paper's k = m+1),
interfaces k = 0..d-2 separating modes <= k | > k.  Interface k holds r_k pivots; pivot slot
s is a full d-tuple PIV[k][s] whose first k+1 entries are the left multi-index I_{<=k}[s]
and whose last d-k-1 entries are the right multi-index I_{>k}[s] (§3.1-3.2,
eq. (3)), plus its parents PAR[k][s] = (alpha, beta): the slot of its left
part in I_{<=k-1} and of its right part in I_{>k+1} (nestedness, eq. (4)).

Pieces (each cites the passage it follows):
  splitmix64 / initial_state -- the first pivot: first argmax |A| over seeded random
                                multi-indices (Alg. 2 line 1 "random set of samples",
                                PAPER.md line 236), rank 1 on every interface.
  superblock_update          -- one step of Alg. 6 (lines 624-641) for superblock k:
                                Alg. 2 (lines 231-253) -- random samples, then rook
                                (column/row partial pivoting) on the error A - A~ of the
                                superblock A(I_{<=k-1} i_k, i_{k+1} I_{>k+1}); the new pivot
                                is appended (Alg. 6 line 4), never swapped, so nestedness is
                                kept (Remark, lines 509-512).
  sweep                      -- Alg. 6 over all superblocks, each reading the index sets of
                                the previous sweep (§3.4 relaxation, lines 599-604).
  integrate                  -- §4.1 "product of (2d-1) matrices" (lines 689-693).

One sweep adds at most one pivot per superblock (Alg. 6 with Alg. 2 applied once); the
workloads run as many sweeps as the rank cap needs (R7).

The cross approximation of a superblock is kept in the incomplete-LU ("ACA") form of the
interpolation formula eq. (1): A~(x, y) = sum_t u_t(x) v_t(y) with
u_t = E_{t-1}(:, y_t), v_t = E_{t-1}(x_t, :) / E_{t-1}(x_t, y_t), which equals
A(:, J) A(I, J)^{-1} A(I, :) (the Schur-complement identity; pinned in the tests).  All sums
over t run t = 0, 1, ... with a separate multiply and subtract (no fused multiply-add);
every argmax takes the FIRST maximiser (numpy semantics).  DESIGN.md R4.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .integrand import X_FAMILIES, entries, prefactor

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
TAG_INIT = 0
N_INIT = 64


def splitmix64(seed: int, ctr: int) -> int:
    """Counter-based splitmix64: mix(seed + (ctr+1)*golden) (Steele et al. 2014)."""
    z = (seed + (ctr + 1) * GOLDEN) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def draw_ctr(tag: int, d: int, i: int, s: int) -> int:
    return ((tag * (d + 1) + i) << 20) + s


def sample_tag(sweep: int) -> int:
    return 1 + sweep


@dataclass
class Problem:
    family: int
    u: np.ndarray          # (d, n) u-nodes
    w: np.ndarray          # (d, n) quadrature weights
    rank_cap: int
    tol: float
    n_samples: int = 32    # |L| of Alg. 2 line 1
    rook_iters: int = 4    # column+row rounds of the rook search (Alg. 2 lines 2-5)
    seed: int = 0
    fold: bool = False     # cross on B = w x ... x w * f (§4.1), x-form

    @property
    def d(self):
        return self.u.shape[0]

    @property
    def n(self):
        return self.u.shape[1]

    @property
    def qw(self):
        """Quadrature weights of the contraction: the rule's weights, or ones when they are
        folded into the tensor (B = w x ... x w * f sums with unit weights)."""
        return np.ones_like(self.w) if self.fold else self.w

    def A(self, idx):
        f = entries(self.family, self.u, idx)
        if not self.fold:
            return f
        # B(i) = f(i) * (((1 * w_0[i_0]) * w_1[i_1]) * ...), this order on both sides
        idx = np.asarray(idx)
        W = np.ones(idx.shape[:-1])
        for j in range(idx.shape[-1]):
            W = W * self.w[j][idx[..., j]]
        return f * W


@dataclass
class State:
    piv: list            # piv[k] : int64 array (r_k, d)   full d-tuples
    par: list            # par[k] : int64 array (r_k, 2)   (alpha, beta) parent slots
    sweep: int = 0
    n_evals: int = 0
    log: list = field(default_factory=list)

    @property
    def ranks(self):
        return [len(p) for p in self.piv]

    def copy(self):
        return State([p.copy() for p in self.piv], [q.copy() for q in self.par], self.sweep, self.n_evals,
                     list(self.log))


def initial_state(prob: Problem) -> State:
    """Rank-1 nested start: t0 = first argmax |A| over N_INIT seeded random multi-indices
    (coordinate j of sample q drawn with counter draw_ctr(TAG_INIT, d, 0, q*d + j))."""
    d, n = prob.d, prob.n
    cand = np.array([[splitmix64(prob.seed, draw_ctr(TAG_INIT, d, 0, q * d + j)) % n for j in range(d)]
                     for q in range(N_INIT)], dtype=np.int64)
    vals = prob.A(cand)
    t0 = cand[int(np.argmax(np.abs(vals)))]
    st = State([t0[None, :].copy() for _ in range(d - 1)], [np.zeros((1, 2), np.int64) for _ in range(d - 1)])
    st.n_evals = N_INIT
    return st


# --------------------------------------------------------------------------------------
# fibers (TT factors of eq. (3) and the quadrature)
# --------------------------------------------------------------------------------------
def fiber(prob: Problem, left_tuples, m, right_tuples):
    """F[alpha][beta][a] = A(left_tuples[alpha][0:m], a, right_tuples[beta][m+1:d]).

    left_tuples / right_tuples are arrays of full d-tuples (only the named parts are
    read); use None for the empty multi-index (m = 0 resp. m = d-1).
    """
    d, n = prob.d, prob.n
    Lt = np.zeros((1, d), np.int64) if left_tuples is None else np.asarray(left_tuples)
    Rt = np.zeros((1, d), np.int64) if right_tuples is None else np.asarray(right_tuples)
    rx, ry = len(Lt), len(Rt)
    idx = np.empty((rx, ry, n, d), dtype=np.int64)
    idx[..., :m] = Lt[:, None, None, :m]
    idx[..., m] = np.arange(n)[None, None, :]
    idx[..., m + 1:] = Rt[None, :, None, m + 1:]
    return prob.A(idx)


# --------------------------------------------------------------------------------------
# one superblock of Alg. 6 (Alg. 2 repeated n_add times)
# --------------------------------------------------------------------------------------
class Superblock:
    """A(I_{<=k-1} i_k, i_{k+1} I_{>k+1}) as an R x C matrix, R = r_{k-1} n, C = n r_{k+1};
    row x = alpha*n + a, column y = beta*n + b (Alg. 3-5 superblock, line 406)."""

    def __init__(self, prob, st, k):
        self.prob, self.k = prob, k
        d, n = prob.d, prob.n
        self.L = st.piv[k - 1] if k > 0 else np.zeros((1, d), np.int64)
        self.Rt = st.piv[k + 1] if k < d - 2 else np.zeros((1, d), np.int64)
        self.R = len(self.L) * n
        self.C = len(self.Rt) * n
        self.evals = 0

    def tuples(self, xs, ys):
        k, n, d = self.k, self.prob.n, self.prob.d
        xs = np.asarray(xs, np.int64)
        ys = np.asarray(ys, np.int64)
        idx = np.empty(xs.shape + (d,), np.int64)
        idx[..., :k] = self.L[xs // n][..., :k]
        idx[..., k] = xs % n
        idx[..., k + 1] = ys % n
        idx[..., k + 2:] = self.Rt[ys // n][..., k + 2:]
        return idx

    def A(self, xs, ys):
        xs, ys = np.broadcast_arrays(np.asarray(xs, np.int64), np.asarray(ys, np.int64))
        self.evals += xs.size
        return self.prob.A(self.tuples(xs, ys))


def _approx_sub(vals, U_rows, V_cols):
    """vals - sum_t U_rows[..., t] * V_cols[..., t], t ascending, mul then sub."""
    out = np.array(vals, dtype=np.float64, copy=True)
    for t in range(U_rows.shape[-1]):
        out = out - U_rows[..., t] * V_cols[..., t]
    return out


def superblock_update(prob: Problem, st: State, k: int):
    """New pivots of interface k from the state of the previous sweep (Alg. 6 line 3).

    Returns (new_piv (r', d), new_par (r', 2), info) with the old pivots first.
    """
    d, n = prob.d, prob.n
    sb = Superblock(prob, st, k)
    R, C = sb.R, sb.C
    P = st.piv[k]
    xs = list(st.par[k][:, 0] * n + P[:, k])
    ys = list(st.par[k][:, 1] * n + P[:, k + 1])
    allx, ally = np.arange(R), np.arange(C)
    U = np.zeros((R, 0))
    V = np.zeros((0, C))

    def col(y, mask):   # (A(:, y), E(:, y)) with E zeroed on the rows in `mask`
        raw = sb.A(allx, y)
        e = _approx_sub(raw, U, np.broadcast_to(V[:, y], (R, V.shape[0])))
        e[mask] = 0.0
        return raw, e

    def row(x, mask):   # (A(x, :), E(x, :)) with E zeroed on the columns in `mask`
        raw = sb.A(x, ally)
        e = _approx_sub(raw, np.broadcast_to(U[x, :], (C, U.shape[1])), V.T)
        e[mask] = 0.0
        return raw, e

    # incomplete LU of the existing cross in slot order (the "LU-pivoted init"): it rebuilds
    # u_s, v_s on the grown superblock exactly as they were when pivot s was added
    scale = 0.0
    for s in range(len(P)):
        raw, c = col(ys[s], xs[:s])
        _, g = row(xs[s], ys[:s])
        if c[xs[s]] == 0.0:
            # singular existing cross: only possible for a zero first pivot, i.e. every
            # seeded sample of A was zero (e.g. D_d with d > n); R8
            info = {"added": 0, "rook_steps": 0, "stop": "singular", "adds": [], "evals": sb.evals,
                    "search_evals": 0, "rank": len(P)}
            return P.copy(), st.par[k].copy(), info
        U = np.concatenate([U, c[:, None]], axis=1)
        V = np.concatenate([V, (g / c[xs[s]])[None, :]], axis=0)
        scale = max(scale, abs(float(raw[xs[s]])))
    new_t, new_p = [], []
    lu_evals = sb.evals
    info = {"added": 0, "rook_steps": 0, "stop": "added", "adds": [], "lu_evals": lu_evals}
    while True:   # one Alg. 2 step (a loop only so that the stop conditions can `break`)
        if len(xs) >= prob.rank_cap:
            info["stop"] = "cap"
            break
        # Alg. 2 line 1: random samples, pick the largest error (pivot rows/columns excluded)
        tag = sample_tag(st.sweep)
        sx = np.array([splitmix64(prob.seed, draw_ctr(tag, d, k, 2 * q)) % R
                       for q in range(prob.n_samples)], np.int64)
        sy = np.array([splitmix64(prob.seed, draw_ctr(tag, d, k, 2 * q + 1)) % C
                       for q in range(prob.n_samples)], np.int64)
        e = _approx_sub(sb.A(sx, sy), U[sx, :], V[:, sy].T)
        e[np.isin(sx, xs) | np.isin(sy, ys)] = 0.0
        q = int(np.argmax(np.abs(e)))
        xst, yst = int(sx[q]), int(sy[q])
        start = (xst, yst)
        # Alg. 2 lines 2-5: rook search -- column partial pivoting, then row partial pivoting,
        # until the row step keeps the column (rook condition eq. (2)) or the budget is spent
        c_at = g_at = -1
        for it in range(prob.rook_iters):
            raw_c, c = col(yst, xs)
            c_at = yst
            xn = int(np.argmax(np.abs(c)))
            _, g = row(xn, ys)
            g_at = xn
            yn = int(np.argmax(np.abs(g)))
            info["rook_steps"] += 1
            conv = yn == yst
            xst, yst = xn, yn
            if conv:
                break
        if c_at != yst:
            raw_c, c = col(yst, xs)
        if g_at != xst:
            _, g = row(xst, ys)
        pv = g[yst]
        if not abs(pv) > prob.tol * scale:
            info["stop"] = "tol"
            break
        xs.append(xst)
        ys.append(yst)
        new_t.append(sb.tuples(np.array([xst]), np.array([yst]))[0])
        new_p.append((xst // n, yst // n))
        info["added"] += 1
        info["adds"].append({"x": xst, "y": yst, "start": start, "pivot": float(pv),
                             "converged": bool(c_at == yst and g_at == xst),
                             "xs_before": list(xs[:-1]), "ys_before": list(ys[:-1])})
        break
    info["evals"] = sb.evals
    info["search_evals"] = sb.evals - lu_evals   # samples + rook columns/rows (Alg. 2)
    info["rank"] = len(xs)
    piv = np.concatenate([P, np.array(new_t, np.int64).reshape(-1, d)], axis=0)
    par = np.concatenate([st.par[k], np.array(new_p, np.int64).reshape(-1, 2)], axis=0)
    return piv, par, info


def sweep(prob: Problem, st: State, interfaces=None) -> State:
    """One dimension-parallel sweep (Alg. 6): every superblock in ``interfaces`` (default:
    all) is updated from ``st``; returns the new state."""
    d = prob.d
    interfaces = range(d - 1) if interfaces is None else interfaces
    new = st.copy()
    infos = {}
    for k in interfaces:
        piv, par, info = superblock_update(prob, st, k)
        new.piv[k], new.par[k] = piv, par
        new.n_evals += info["evals"]
        infos[k] = info
    new.log.append((st.sweep, infos))
    new.sweep = st.sweep + 1
    return new


# --------------------------------------------------------------------------------------
# TT quadrature (§4.1)
# --------------------------------------------------------------------------------------
def intersection(prob, state, i):
    """M_i = A(I_{<=i}, I_{>i}):  M[s, t] = A(left(PIV[i][s]), right(PIV[i][t]))."""
    P = state.piv[i]
    r = len(P)
    idx = np.empty((r, r, prob.d), dtype=np.int64)
    idx[..., :i + 1] = P[:, None, :i + 1]
    idx[..., i + 1:] = P[None, :, i + 1:]
    return prob.A(idx)


def tt_fibers(prob, state):
    d = prob.d
    return [fiber(prob, state.piv[m - 1] if m > 0 else None, m,
                  state.piv[m] if m < d - 1 else None) for m in range(d)]


def integrate(prob, state, fibers=None):
    """I = (4/d!) * W_0 M_0^{-1} W_1 M_1^{-1} ... W_{d-1},  W_m = sum_a w_{m,a} F_m[:,:,a].

    The row vector is renormalised by its max-abs after every factor (exact log2
    bookkeeping) so that d = 200 neither overflows nor underflows.
    Returns (value, log10|value|, sign, n_evals).
    """
    d = prob.d
    fibers = tt_fibers(prob, state) if fibers is None else fibers
    n_evals = sum(F.size for F in fibers)
    log2s = 0.0
    v = None
    for m in range(d):
        W = fibers[m] @ prob.qw[m]                     # (r_{m-1}, r_m)
        v = W[0] if v is None else v @ W
        if m < d - 1:
            M = intersection(prob, state, m)
            n_evals += M.size
            v = np.linalg.solve(M.T, v)
        mx = float(np.max(np.abs(v)))
        if mx == 0.0 or not np.isfinite(mx):
            break
        ex = math.frexp(mx)[1]
        v = np.ldexp(v, -ex)
        log2s += ex
    core = float(v[0]) if v is not None and v.size else 0.0
    sign = 1 if core > 0 else (-1 if core < 0 else 0)
    if core == 0.0 or not math.isfinite(core):
        return core, -math.inf if core == 0.0 else math.nan, sign, n_evals
    xform = prob.family in X_FAMILIES
    lnpre = math.log(2.0) if xform else math.log(4.0) - math.lgamma(d + 1)
    ln_abs = math.log(abs(core)) + log2s * math.log(2.0) + lnpre
    log10 = ln_abs / math.log(10.0)
    if -700.0 < ln_abs < 700.0:
        # direct product when every factor is representable (keeps full fp64 accuracy)
        if -1000 < log2s < 1000 and (xform or d <= 170):
            value = math.ldexp(core, int(log2s)) * prefactor(d, prob.family)
        else:
            value = sign * math.exp(ln_abs)
    else:
        value = sign * (math.inf if ln_abs > 0 else 0.0)
    return value, log10, sign, n_evals


def _dd_weighted_sum(F, w):
    """sum_a w_a F[..., a] in double-double (Dekker products, Knuth sums), vectorised."""
    from .integrand import _two_prod
    hi = np.zeros(F.shape[:-1])
    lo = np.zeros(F.shape[:-1])
    for a in range(F.shape[-1]):
        p, e = _two_prod(np.full(hi.shape, w[a]), F[..., a])
        s = hi + p
        bb = s - hi
        err = (hi - (s - bb)) + (p - bb)
        lo = lo + err + e
        hi = s + lo
        lo = lo - (hi - s)
    return hi, lo


def integrate_exact(prob, state, fibers=None, dps=50):
    """The §4.1 product (4/d!) W_0 M_0^{-1} ... W_{d-1} evaluated (nearly) exactly for the
    given fp64 fiber entries: W sums in double-double, the chain in mpmath at ``dps``
    digits.  DESIGN.md R9: this -- not the fp64 evaluation, whose error grows like
    cond(M_i) * eps -- is what the CUDA path's double-double contraction is compared with.
    Returns (value, log10|value|, sign)."""
    import mpmath
    d = prob.d
    fibers = tt_fibers(prob, state) if fibers is None else fibers
    with mpmath.workdps(dps):
        v = None
        for m in range(d):
            hi, lo = _dd_weighted_sum(fibers[m], prob.qw[m])
            W = mpmath.matrix(hi.shape[0], hi.shape[1])
            for a in range(hi.shape[0]):
                for b in range(hi.shape[1]):
                    W[a, b] = mpmath.mpf(float(hi[a, b])) + mpmath.mpf(float(lo[a, b]))
            v = W[0, :] if v is None else v * W
            if m < d - 1:
                M = mpmath.matrix(intersection(prob, state, m).tolist())
                v = mpmath.lu_solve(M.T, v.T).T
        core = v[0]
        if core == 0:
            return 0.0, -math.inf, 0
        sign = 1 if core > 0 else -1
        val = core * 2 if prob.family in X_FAMILIES else core * 4 / mpmath.factorial(d)
        return float(val), float(mpmath.log10(abs(val))), sign


def run(prob, n_sweeps, state=None):
    """Init (if no state), n_sweeps sweeps, then the quadrature."""
    st = initial_state(prob) if state is None else state
    for _ in range(n_sweeps):
        st = sweep(prob, st)
    val, log10, sign, ev = integrate(prob, st)
    st.n_evals += ev
    return st, val, log10
