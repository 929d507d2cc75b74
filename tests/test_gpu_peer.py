"""The cross-GPU wavefront's exchange code (include/ttcross.h: tt_cross_sweep_peer), run on one
GPU through the loopback of tt_cross_set_loopback.

The interfaces are split at a boundary b as if [0, b) and [b, d-1) lived on two ranks: in the
ONE persistent launch of tt_cross_sweep, superblocks b-1 and b publish their new record, rank
and done flag into a mirror buffer with the code a rank's boundary superblocks use for the
neighbour rank's peer memory (plain stores + a system-scope release), and each waits on the
other's mirror flag with a system-scope acquire.  Nothing waits on another launch, so this is
safe on one device.  Checks: the pivots are bit-identical to the plain solve after every
sweep (Alg. 6: the sweep reads only the neighbours' pivots of the previous sweep),
the integral is the same bits, and the mirror holds exactly what a neighbour rank must receive
-- the boundary interfaces' records, their rank after the last sweep and their done count.
"""
import numpy as np
import pytest

from workloads import FAMILY_C, FAMILY_D, WORKLOADS, ising_grid

pytestmark = pytest.mark.gpu


def _solve(tt, sweeps, per_sweep):
    states = []
    if per_sweep:
        for _ in range(sweeps):
            tt.sweep(1)
            states.append(tt.state(parents=True))
    else:
        tt.sweep(sweeps)
        states.append(tt.state(parents=True))
    return states, tt.integrate()


def _check_mirror(tt, b, sweeps, ranks, piv, par):
    rec, ring, done = tt.loopback()
    d, cap = tt.d, tt.cap
    for k in (b - 1, b):   # the boundary superblocks: their records went through the peer path
        r = int(ranks[k])
        assert rec[k, 0] == r, f"interface {k}: mirror rank word {rec[k, 0]} != {r}"
        tup = rec[k, 1:1 + r * d].reshape(r, d)
        pr = rec[k, 1 + cap * d:1 + cap * d + 2 * r].reshape(r, 2)
        assert np.array_equal(tup, piv[k]), f"interface {k}: mirror tuples differ"
        assert np.array_equal(pr, par[k]), f"interface {k}: mirror parents differ"
        assert ring[k, (sweeps - 1) & 1] == r, f"interface {k}: mirror rank ring"
        assert done[k] == sweeps, f"interface {k}: mirror done flag {done[k]} != {sweeps}"
    others = [k for k in range(d - 1) if k not in (b - 1, b)]
    assert all(done[k] == 0 for k in others), "only the boundary superblocks publish to a neighbour rank"


@pytest.mark.parametrize("family,d,n,L,cap,sweeps,b", [
    (FAMILY_C, 6, 33, 8.0, 8, 8, 2),
    (FAMILY_D, 5, 17, 6.0, 8, 8, 1),     # boundary at the first interface
    (FAMILY_D, 7, 21, 6.0, 6, 6, 5),     # ... at the last
    (FAMILY_C, 9, 65, 10.0, 12, 10, 4),
])
def test_loopback_equals_single(lib, family, d, n, L, cap, sweeps, b):
    from paper_1903_11554_b200 import TTCross
    u, w = ising_grid(d, n, L)
    ref = TTCross(family, u, w, cap, 1e-12, n_samples=16, rook_iters=4, seed=3)
    if not ref.launch_shape()["persistent"]:
        pytest.skip("no persistent launch for this shape")
    rs, rv = _solve(ref, sweeps, True)
    tt = TTCross(family, u, w, cap, 1e-12, n_samples=16, rook_iters=4, seed=3)
    tt.set_loopback(b)
    ls, lv = _solve(tt, sweeps, True)
    for s in range(sweeps):
        assert list(rs[s][0]) == list(ls[s][0]), f"sweep {s}: ranks differ"
        for x, y in zip(rs[s][1] + rs[s][2], ls[s][1] + ls[s][2]):
            assert np.array_equal(x, y), f"sweep {s}: loopback pivots differ"
    assert lv == rv, "integral differs"
    _check_mirror(tt, b, sweeps, *ls[-1])
    # off again: the plain path, same result
    tt.set_loopback(0)
    os_, ov = _solve(tt, sweeps, False)
    assert ov == rv
    ref.close()
    tt.close()


@pytest.mark.parametrize("name,b", [("D5", 2), ("C10", 4), ("D20", 9), ("C200", 100)])
def test_loopback_workloads_one_launch(lib, name, b):
    """The BASELINE configs (the streaming shapes of D_20 / C_200 included): all Alg. 6 sweeps
    in one persistent launch with the loopback boundary in the middle, bit-identical to the
    plain solve."""
    from paper_1903_11554_b200 import TTCross
    wl = WORKLOADS[name]
    u, w = wl.grid()
    kw = dict(n_samples=wl.n_samples, rook_iters=wl.rook_iters, seed=wl.seed)
    ref = TTCross(wl.family, u, w, wl.rank_cap, wl.tol, **kw)
    shape = ref.launch_shape()
    assert shape["persistent"] and shape["all_resident"], "the BASELINE configs run the (cross-GPU) wavefront"
    rs, rv = _solve(ref, wl.alg6_sweeps, False)
    tt = TTCross(wl.family, u, w, wl.rank_cap, wl.tol, **kw)
    tt.set_loopback(b)
    ls, lv = _solve(tt, wl.alg6_sweeps, False)
    assert list(rs[0][0]) == list(ls[0][0])
    for x, y in zip(rs[0][1] + rs[0][2], ls[0][1] + ls[0][2]):
        assert np.array_equal(x, y), "loopback pivots differ"
    assert lv == rv
    _check_mirror(tt, b, wl.alg6_sweeps, *ls[0])
    ref.close()
    tt.close()


def test_peer_entry_points_reject_world_one(lib):
    from paper_1903_11554_b200 import TTCross
    from paper_1903_11554_b200.binding import TTCError
    u, w = ising_grid(5, 17, 6.0)
    tt = TTCross(FAMILY_D, u, w, 8, 1e-12, n_samples=16, rook_iters=4, seed=3)
    with pytest.raises(TTCError):
        tt.peer_handles()
    with pytest.raises(TTCError):
        tt.sweep_peer(1)
    with pytest.raises(TTCError):
        tt.set_loopback(4)          # outside [1, d-2]
    with pytest.raises(TTCError):
        tt.loopback()               # loopback off
    tt.close()
