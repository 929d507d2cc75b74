"""Multi-process host logic of the dimension-parallel cross on CPU (gloo, world_size 2).

What is checked: the superblock partition rule (Alg. 6 line 1) matches the one the
library uses (exchange-buffer size); the record encoding round-trips; and a 2-process run
of Alg. 6 -- each rank updates only its own superblocks (with the oracle standing in for
the device work), packs them into the exchange-buffer layout, all-gathers with
`allgather_slices`, unpacks -- gives exactly the single-process sweep, sweep after sweep.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cross as X
from paper_1903_11554_b200.dist import (allgather_slices, owned_interfaces, pack_records, pack_slots,
                                        record_stride, unpack_records, unpack_slots)
from workloads import FAMILY_C, FAMILY_D, ising_grid


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("d,world", [(2, 1), (5, 2), (6, 4), (200, 8), (3, 8)])
def test_partition_covers_every_interface_once(d, world):
    seen = []
    for r in range(world):
        kb, ke, chunk = owned_interfaces(d, r, world)
        assert 0 <= kb <= ke <= d - 1 and ke - kb <= chunk
        seen += list(range(kb, ke))
    assert seen == list(range(d - 1))


def test_partition_is_balanced():
    """Alg. 6 line 1 with balanced blocks: shares differ by at most one, larger first."""
    shares = [owned_interfaces(20, r, 8)[1] - owned_interfaces(20, r, 8)[0] for r in range(8)]
    assert shares == [3, 3, 3, 2, 2, 2, 2, 2]
    shares = [owned_interfaces(200, r, 8)[1] - owned_interfaces(200, r, 8)[0] for r in range(8)]
    assert shares == [25, 25, 25, 25, 25, 25, 25, 24]
    assert [owned_interfaces(3, r, 4)[1] - owned_interfaces(3, r, 4)[0] for r in range(4)] == [1, 1, 0, 0]
    for d in (2, 5, 20, 201):
        for world in (1, 2, 3, 8):
            sh = [owned_interfaces(d, r, world)[1] - owned_interfaces(d, r, world)[0] for r in range(world)]
            assert max(sh) - min(sh) <= 1 and sh == sorted(sh, reverse=True) and max(sh) <= owned_interfaces(d, 0, world)[2]


def test_record_roundtrip():
    prob = X.Problem(FAMILY_D, *ising_grid(5, 9, 3.0), 6, 1e-12, 16, 4, 3)
    st = X.initial_state(prob)
    for _ in range(4):
        st = X.sweep(prob, st)
    buf = pack_records(st.piv, st.par, 5, 6, 4)
    assert buf.numel() == 4 * record_stride(5, 6)
    piv, par = unpack_records(buf, 5, 6, 4)
    for k in range(4):
        assert np.array_equal(piv[k].numpy(), st.piv[k]) and np.array_equal(par[k].numpy(), st.par[k])


def _worker(rank, world, port, d, n, cap, sweeps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        u, w = ising_grid(d, n, 4.0)
        prob = X.Problem(FAMILY_C, u, w, cap, 1e-12, 16, 4, 5)
        kb, ke, chunk = owned_interfaces(d, rank, world)
        rs = record_stride(d, cap)
        st = X.initial_state(prob)
        for _ in range(sweeps):
            mine = X.sweep(prob, st, range(kb, ke))          # this rank's superblocks only
            local = pack_records(mine.piv, mine.par, d, cap, d - 1)
            xbuf = pack_slots(local, d, cap, world)          # own records -> own slot
            allgather_slices(xbuf, chunk * rs)                # the exchange of Alg. 6 lines 6-8
            rec = unpack_slots(xbuf, pack_records(st.piv, st.par, d, cap, d - 1), d, cap, world)
            piv, par = unpack_records(rec, d, cap, d - 1)
            st = X.State([p.numpy() for p in piv], [p.numpy() for p in par], st.sweep + 1, 0)
        if rank == 0:
            q.put([p.tolist() for p in st.piv])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("d,world", [(6, 2), (5, 2), (7, 3)])
def test_two_process_sweeps_equal_single_process(d, world):
    n, cap, sweeps = 7, 5, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, d, n, cap, sweeps, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    u, w = ising_grid(d, n, 4.0)
    prob = X.Problem(FAMILY_C, u, w, cap, 1e-12, 16, 4, 5)
    st = X.initial_state(prob)
    for _ in range(sweeps):
        st = X.sweep(prob, st)
    assert [p.tolist() for p in st.piv] == got


def test_neighbour_handles_chain():
    """tt_cross_peer_open's contract: rank p gets rank p-1's handles on the left and rank p+1's
    on the right, None at the ends of the chain (Alg. 6 lines 6-8: neighbours only)."""
    from paper_1903_11554_b200.dist import neighbour_handles
    hs = [bytes([p]) * 4 for p in range(4)]
    assert neighbour_handles(hs, 0, 4) == (None, hs[1])
    assert neighbour_handles(hs, 2, 4) == (hs[1], hs[3])
    assert neighbour_handles(hs, 3, 4) == (hs[2], None)
    assert neighbour_handles(hs[:1], 0, 1) == (None, None)
    with pytest.raises(ValueError):
        neighbour_handles(hs, 0, 3)
