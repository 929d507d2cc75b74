"""The partitioned (multi-GPU) path of the library, emulated in one process on one GPU.

Two contexts with world = 2 (rank 0 and rank 1) each update only their own superblocks
(tt_cross_sweep_local); the all-gather of PAPER.md Alg. 6 lines 6-8 is emulated by copying
each rank's slice of its exchange buffer into the other rank's buffer (what
paper_1903_11554_b200.dist does with NCCL), then both commit.  Nothing waits on another
launch, so this is safe on one device.  The result must equal the single-context solve:
pivots bit-exact after every sweep; the integral, whose chain product is split at the rank
boundary, within double-double rounding.
"""
import numpy as np
import pytest

from workloads import FAMILY_C, FAMILY_D, WORKLOADS, ising_grid

pytestmark = pytest.mark.gpu


def exchange(views, per_rank_elems):
    import torch
    bufs = [torch.as_tensor(v, device="cuda") for v in views]
    world = len(bufs)
    for src in range(world):
        sl = slice(src * per_rank_elems, (src + 1) * per_rank_elems)
        for dst in range(world):
            if dst != src:
                bufs[dst][sl].copy_(bufs[src][sl])
    torch.cuda.synchronize()


def run_partitioned(family, u, w, cap, tol, ns, rook, seed, sweeps, world, fold=False):
    from paper_1903_11554_b200 import TTCross
    tts = [TTCross(family, u, w, cap, tol, n_samples=ns, rook_iters=rook, seed=seed, rank=p, world=world,
                   fold_weights=fold) for p in range(world)]
    xv = [t.exchange_view() for t in tts]
    per = xv[0][1] // 4
    states = []
    for _ in range(sweeps):
        for t in tts:
            t.sweep_local()
        exchange([v for v, _ in xv], per)
        for t in tts:
            t.commit()
        states.append(tts[0].state(parents=True))
        for t in tts[1:]:
            other = t.state(parents=True)
            for a, b in zip(states[-1][1] + states[-1][2], other[1] + other[2]):
                assert np.array_equal(a, b), "ranks disagree on the committed pivots"
    for t in tts:
        t.integrate_local()
    pv = [t.partials_view() for t in tts]
    exchange([v for v, _ in pv], pv[0][1] // 8)
    val = tts[0].integrate_finish()
    for t in tts:
        t.close()
    return states, val


@pytest.mark.parametrize("family,d,n,L,cap,sweeps,world", [
    (FAMILY_C, 6, 33, 8.0, 8, 8, 2),
    (FAMILY_D, 5, 17, 6.0, 8, 8, 2),
    (FAMILY_D, 7, 21, 6.0, 6, 6, 3),    # uneven chunks
    (FAMILY_C, 4, 17, 6.0, 5, 5, 4),    # a rank owning no superblock
])
def test_partitioned_equals_single(lib, family, d, n, L, cap, sweeps, world):
    from paper_1903_11554_b200 import TTCross
    u, w = ising_grid(d, n, L)
    states, val = run_partitioned(family, u, w, cap, 1e-12, 16, 4, 3, sweeps, world)
    ref = TTCross(family, u, w, cap, 1e-12, n_samples=16, rook_iters=4, seed=3)
    for s in range(sweeps):
        ref.sweep(1)
        r = ref.state(parents=True)
        assert list(r[0]) == list(states[s][0])
        for a, b in zip(r[1] + r[2], states[s][1] + states[s][2]):
            assert np.array_equal(a, b), f"sweep {s}: partitioned pivots differ"
    rv = ref.integrate()
    assert val[2] == rv[2]
    assert abs(val[0] - rv[0]) <= 1e-13 * abs(rv[0])
    ref.close()


def test_partitioned_d5_workload(lib):
    wl = WORKLOADS["D5"]
    u, w = wl.grid()
    from paper_1903_11554_b200 import TTCross
    states, val = run_partitioned(wl.family, u, w, wl.rank_cap, wl.tol, wl.n_samples, wl.rook_iters, wl.seed,
                                  wl.alg6_sweeps, 2)
    ref = TTCross(wl.family, u, w, wl.rank_cap, wl.tol, n_samples=wl.n_samples, rook_iters=wl.rook_iters,
                  seed=wl.seed)
    ref.sweep(wl.alg6_sweeps)
    r = ref.state(parents=True)
    for a, b in zip(r[1] + r[2], states[-1][1] + states[-1][2]):
        assert np.array_equal(a, b)
    rv = ref.integrate()
    assert abs(val[0] - rv[0]) <= 1e-13 * abs(rv[0])
    ref.close()


@pytest.mark.parametrize("fold", [False, True])
def test_partitioned_xform(lib, fold):
    """The x-form path (direct entries, optional folded weights) partitioned over 3 ranks."""
    from paper_1903_11554_b200 import TTCross
    from workloads import FAMILY_DX, xform_grid
    x, w = xform_grid(7, 13)
    states, val = run_partitioned(FAMILY_DX, x, w, 6, 1e-14, 16, 4, 9, 6, 3, fold)
    ref = TTCross(FAMILY_DX, x, w, 6, 1e-14, n_samples=16, rook_iters=4, seed=9, fold_weights=fold)
    ref.sweep(6)
    r = ref.state(parents=True)
    for a, b in zip(r[1] + r[2], states[-1][1] + states[-1][2]):
        assert np.array_equal(a, b)
    rv = ref.integrate()
    assert abs(val[0] - rv[0]) <= 1e-13 * abs(rv[0])
    ref.close()
