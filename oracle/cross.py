"""ORACLE (test infrastructure only): dimension-parallel TT cross + TT quadrature.

Follows DESIGN.md §2 (the method) step by step.  Notation: modes m = 0..d-1 (paper's
k = m+1), interfaces i = 0..d-2 separating modes <= i | > i.  The cross state is, for every
interface i, r_i pivots; pivot slot s is a full d-tuple PIV[i][s] whose first i+1 entries
are the left multi-index I_{<=i}[s] and whose last d-i-1 entries are the right multi-index
I_{>i}[s] (§3.1-3.2, eq. (3)).

Pieces (each cites the passage it follows):
  splitmix64 / initial_state  -- seed-fixed random nested initial pivots (BASELINE.json
                                 "seed-fixed random initial pivots"; nestedness eq. (4)).
  enrich_right / enrich_left  -- random extra candidate columns of the superblock
                                 (Alg. 2 line 1 "Pick a random set of samples", PAPER.md
                                 lines 236-240, applied to whole superblock columns).
  fiber                       -- A(I_{<=m-1}, i_m, I_{>m}) as an array [alpha][beta][a]
                                 (eq. (3) factors, lines 314-320).
  rrcross                     -- rank-revealing cross of a fiber matrix by complete
                                 pivoting (§2.4: "complete pivoting ...
                                 numerically stable") with truncation at tol and the
                                 rank cap, maintaining B = A(:,J) A(I,J)^{-1}.
  maxvol                      -- Alg. 1 (lines 205-218) iterated: swap while
                                 max|B| > 1 + delta, with the rank-1 update of B from
                                 the paper's maxvol reference [gostz-maxvol-2010].
  half_sweep                  -- Alg. 3 directions with the dimension-parallel
                                 relaxation of §3.4 (lines 599-604): every interface is
                                 updated from the index sets of the previous half-sweep.
  integrate                   -- §4.1 "product of (2d-1) matrices" (lines 689-693).

All argmax decisions take the FIRST maximiser in row-major order (numpy semantics).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .integrand import entries, prefactor

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
TAG_INIT_LEFT = 0
TAG_INIT_RIGHT = 1
DIR_LR = 0
DIR_RL = 1


def splitmix64(seed: int, ctr: int) -> int:
    """Counter-based splitmix64: mix(seed + (ctr+1)*golden) (Steele et al. 2014)."""
    z = (seed + (ctr + 1) * GOLDEN) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def draw_ctr(tag: int, d: int, i: int, s: int) -> int:
    return ((tag * (d + 1) + i) << 20) + s


def enrich_tag(sweep: int, direction: int) -> int:
    return 2 + 2 * sweep + direction


def partial_fisher_yates(seed, tag, d, i, M, r):
    """First r entries of a seeded Fisher-Yates shuffle of range(M) (sparse perm)."""
    perm = {}
    out = []
    for s in range(r):
        j = s + splitmix64(seed, draw_ctr(tag, d, i, s)) % (M - s)
        vs, vj = perm.get(s, s), perm.get(j, j)
        perm[s], perm[j] = vj, vs
        out.append(vj)
    return out


@dataclass
class Problem:
    family: int
    u: np.ndarray          # (d, n) u-nodes
    w: np.ndarray          # (d, n) quadrature weights
    rank_cap: int
    tol: float
    n_enrich: int = 4
    delta: float = 1e-2
    max_swaps: int = 0     # 0 -> 2*rank_cap
    seed: int = 0

    @property
    def d(self):
        return self.u.shape[0]

    @property
    def n(self):
        return self.u.shape[1]

    def swaps_cap(self):
        return self.max_swaps if self.max_swaps > 0 else 2 * self.rank_cap

    def A(self, idx):
        return entries(self.family, self.u, idx)


@dataclass
class State:
    piv: list            # piv[i] : int64 array (r_i, d)
    sweep: int = 0
    n_evals: int = 0
    log: list = field(default_factory=list)

    @property
    def ranks(self):
        return [len(p) for p in self.piv]

    def copy(self):
        return State([p.copy() for p in self.piv], self.sweep, self.n_evals, list(self.log))


def initial_ranks(d, n, cap):
    """r_i = min(cap, n^(i+1), n^(d-1-i)) (a rank can exceed neither unfolding side)."""
    out = []
    for i in range(d - 1):
        out.append(int(min(cap, n ** min(i + 1, 64), n ** min(d - 1 - i, 64))))
    return out


def initial_state(prob: Problem) -> State:
    """Seed-fixed random nested pivots (nestedness eq. (4)).

    Left parts: I_{<=i} = r_i distinct draws from I_{<=i-1} x {0..n-1}, candidate
    c = alpha*n + a -> (I_{<=i-1}[alpha], a).  Right parts: I_{>i} = r_i distinct draws
    from {0..n-1} x I_{>i+1}, candidate c = beta*n + a -> (a, I_{>i+1}[beta]).
    Slot s pairs the s-th left draw with the s-th right draw.
    """
    d, n = prob.d, prob.n
    r = initial_ranks(d, n, prob.rank_cap)
    left = []
    for i in range(d - 1):
        prev = r[i - 1] if i > 0 else 1
        sel = partial_fisher_yates(prob.seed, TAG_INIT_LEFT, d, i, prev * n, r[i])
        rows = []
        for c in sel:
            alpha, a = divmod(c, n)
            rows.append((list(left[i - 1][alpha]) if i > 0 else []) + [a])
        left.append(rows)
    right = [None] * (d - 1)
    for i in range(d - 2, -1, -1):
        nxt = r[i + 1] if i < d - 2 else 1
        sel = partial_fisher_yates(prob.seed, TAG_INIT_RIGHT, d, i, nxt * n, r[i])
        rows = []
        for c in sel:
            beta, a = divmod(c, n)
            rows.append([a] + (list(right[i + 1][beta]) if i < d - 2 else []))
        right[i] = rows
    piv = [np.array([left[i][s] + right[i][s] for s in range(r[i])], dtype=np.int64)
           for i in range(d - 1)]
    return State(piv)


# --------------------------------------------------------------------------------------
# fibers
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


def fiber_matrix(F, direction):
    """Row-major matrix view of a fiber for the given half-sweep direction.

    L->R: rows (alpha, a) -> alpha*n + a, columns beta.
    R->L: rows (beta, a)  -> beta*n + a,  columns alpha.
    """
    rx, ry, n = F.shape
    if direction == DIR_LR:
        return F.transpose(0, 2, 1).reshape(rx * n, ry)
    return F.transpose(1, 2, 0).reshape(ry * n, rx)


# --------------------------------------------------------------------------------------
# rank-revealing cross (complete pivoting) + maxvol
# --------------------------------------------------------------------------------------
def rrcross(F, tol, cap):
    """Complete-pivoting cross of the m x c matrix F with truncation.

    Step: (i, col) = first argmax of |R| (pivoted rows/columns are exactly zero);
    stop if not |R[i,col]| > tol * max|F| or cap pivots were taken.
    Updates (all elementwise, no fused multiply-add):
        b      = R[:, col] / piv
        B      = B - outer(b, B[i, :]),   then append b as the new column
        R      = R - outer(R[:, col], R[i, :] / piv),  R[i,:] = 0, R[:,col] = 0
    Returns (I, J, B) with B = F[:, J] F[I, J]^{-1} (slot order = pivot order).
    An all-zero F returns empty I, J.
    """
    F = np.asarray(F, dtype=np.float64)
    m, c = F.shape
    R = F.copy()
    scale = float(np.max(np.abs(F))) if F.size else 0.0
    B = np.zeros((m, 0))
    I, J = [], []
    for _ in range(min(cap, m, c)):
        flat = int(np.argmax(np.abs(R)))
        i, col = divmod(flat, c)
        piv = R[i, col]
        if not abs(piv) > tol * scale:
            break
        b = R[:, col] / piv
        if B.shape[1]:
            B = B - np.multiply.outer(b, B[i, :])
        B = np.concatenate([B, b[:, None]], axis=1)
        R = R - np.multiply.outer(R[:, col], R[i, :] / piv)
        R[i, :] = 0.0
        R[:, col] = 0.0
        I.append(i)
        J.append(col)
    return I, J, B


def maxvol(B, I, delta, max_swaps):
    """Alg. 1 iterated on B = A(:,J) A(I,J)^{-1}.

    (i, j) = first argmax |B|; stop unless |B[i,j]| > 1 + delta; otherwise I[j] <- i and
        g = (B[i, :] - e_j) / B[i, j];   B = B - outer(B[:, j], g).
    Returns (I, B, n_swaps).
    """
    I = list(I)
    B = B.copy()
    r = B.shape[1]
    nsw = 0
    while nsw < max_swaps and r > 0:
        flat = int(np.argmax(np.abs(B)))
        i, j = divmod(flat, r)
        piv = B[i, j]
        if not abs(piv) > 1.0 + delta:
            break
        e = B[i, :].copy()
        e[j] = e[j] - 1.0
        g = e / piv
        B = B - np.multiply.outer(B[:, j], g)
        I[j] = i
        nsw += 1
    return I, B, nsw


# --------------------------------------------------------------------------------------
# enrichment (random superblock columns)
# --------------------------------------------------------------------------------------
def enrich_right(prob, state, i, sweep):
    """Extended column set of interface i for L->R: existing right parts plus n_enrich
    random (a, I_{>i+1}[beta]) candidates, duplicates (vs everything so far) skipped."""
    d, n = prob.d, prob.n
    ext = [row.copy() for row in state.piv[i]]
    nxt = len(state.piv[i + 1]) if i < d - 2 else 1
    M = nxt * n
    for jdraw in range(prob.n_enrich):
        c = splitmix64(prob.seed, draw_ctr(enrich_tag(sweep, DIR_LR), d, i, jdraw)) % M
        beta, a = divmod(c, n)
        t = np.zeros(d, np.int64)
        t[:i + 1] = -1
        t[i + 1] = a
        if i < d - 2:
            t[i + 2:] = state.piv[i + 1][beta][i + 2:]
        if any(np.array_equal(t[i + 1:], e[i + 1:]) for e in ext):
            continue
        ext.append(t)
    return np.array(ext, dtype=np.int64)


def enrich_left(prob, state, i, sweep):
    """Extended column set of interface i for R->L: existing left parts plus n_enrich
    random (I_{<=i-1}[alpha], a) candidates, duplicates skipped."""
    d, n = prob.d, prob.n
    ext = [row.copy() for row in state.piv[i]]
    prv = len(state.piv[i - 1]) if i > 0 else 1
    M = prv * n
    for jdraw in range(prob.n_enrich):
        c = splitmix64(prob.seed, draw_ctr(enrich_tag(sweep, DIR_RL), d, i, jdraw)) % M
        alpha, a = divmod(c, n)
        t = np.zeros(d, np.int64)
        t[i + 1:] = -1
        if i > 0:
            t[:i] = state.piv[i - 1][alpha][:i]
        t[i] = a
        if any(np.array_equal(t[:i + 1], e[:i + 1]) for e in ext):
            continue
        ext.append(t)
    return np.array(ext, dtype=np.int64)


# --------------------------------------------------------------------------------------
# half-sweeps (dimension parallel) and full sweeps
# --------------------------------------------------------------------------------------
def update_interface(prob, state, i, direction):
    """New pivots of interface i from the state of the previous half-sweep.

    Returns (new_piv_i or None if the fiber is identically zero, info dict).
    """
    d, n = prob.d, prob.n
    if direction == DIR_LR:
        m = i
        X = state.piv[i - 1] if i > 0 else None
        Y = enrich_right(prob, state, i, state.sweep)
    else:
        m = i + 1
        X = enrich_left(prob, state, i, state.sweep)
        Y = state.piv[i + 1] if i + 1 < d - 1 else None
    F = fiber(prob, X, m, Y)
    Fm = fiber_matrix(F, direction)
    I, J, B = rrcross(Fm, prob.tol, prob.rank_cap)
    info = {"evals": F.size, "rank": len(I), "swaps": 0, "cols": Fm.shape[1], "rows": Fm.shape[0]}
    if not I:
        return None, info
    I, B, nsw = maxvol(B, I, prob.delta, prob.swaps_cap())
    info["swaps"] = nsw
    new = np.empty((len(I), d), dtype=np.int64)
    for s, (row, col) in enumerate(zip(I, J)):
        outer, a = divmod(row, n)
        x, y = (outer, col) if direction == DIR_LR else (col, outer)
        if m > 0:
            new[s, :m] = X[x][:m]
        new[s, m] = a
        if m < d - 1:
            new[s, m + 1:] = Y[y][m + 1:]
    return new, info


def half_sweep(prob, state, direction, interfaces=None):
    """One dimension-parallel half-sweep (Alg. 6 lines 2-5 with the §3.4 relaxation).

    Every interface in ``interfaces`` (default: all) is updated from ``state`` (the sets
    of the previous half-sweep); returns the new state (interfaces not listed, or whose
    fiber is identically zero, keep their pivots).
    """
    d = prob.d
    interfaces = range(d - 1) if interfaces is None else interfaces
    new = state.copy()
    infos = {}
    for i in interfaces:
        piv, info = update_interface(prob, state, i, direction)
        if piv is not None:
            new.piv[i] = piv
        new.n_evals += info["evals"]
        infos[i] = info
    new.log.append((state.sweep, direction, infos))
    return new


def sweep(prob, state):
    """One full sweep = L->R half-sweep then R->L half-sweep."""
    s = half_sweep(prob, state, DIR_LR)
    s = half_sweep(prob, s, DIR_RL)
    s.sweep = state.sweep + 1
    return s


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
        W = fibers[m] @ prob.w[m]                      # (r_{m-1}, r_m)
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
    lnpre = math.log(4.0) - math.lgamma(d + 1)
    ln_abs = math.log(abs(core)) + log2s * math.log(2.0) + lnpre
    log10 = ln_abs / math.log(10.0)
    if -700.0 < ln_abs < 700.0:
        # direct product when every factor is representable (keeps full fp64 accuracy)
        if -1000 < log2s < 1000 and d <= 170:
            value = math.ldexp(core, int(log2s)) * prefactor(d)
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
            hi, lo = _dd_weighted_sum(fibers[m], prob.w[m])
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
        val = core * 4 / mpmath.factorial(d)
        return float(val), float(mpmath.log10(abs(val))), sign


def run(prob, n_sweeps, state=None):
    """Init (if no state), n_sweeps full sweeps, then the quadrature."""
    st = initial_state(prob) if state is None else state
    for _ in range(n_sweeps):
        st = sweep(prob, st)
    val, log10, sign, ev = integrate(prob, st)
    st.n_evals += ev
    return st, val, log10
