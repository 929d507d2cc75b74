"""Multi-GPU plumbing of the dimension-parallel TT cross (Alg. 6).

One process per GPU.  Interfaces (superblocks) are partitioned into balanced contiguous
blocks, rank p owning [kb_p, kb_{p+1}) with kb_p = p*q + min(p, m), q = (d-1) // world,
m = (d-1) % world (Alg. 6 line 1 "Deduce the range [k_beg, k_end) of superblocks belonging
to the process p"): D_20 on 8 ranks owns 3,3,3,2,2,2,2,2.  After every sweep each rank has
the new pivots of its own interfaces in its slot of the library's exchange buffer (slots of
chunk = ceil((d-1)/world) records); an all-gather of the slots gives every rank the complete
new index sets (the paper exchanges only neighbour pivots, Alg. 6 lines 6-8; an all-gather
over NVSwitch costs one latency-bound collective of a few KB, and every rank needs the full
sets at the quadrature).  The quadrature all-gathers the per-rank partial chain products
(§4.1: the product of 2d-1 matrices, split at the chunk boundaries)
and multiplies them in rank order.

Everything here is argument marshalling and collectives; the arithmetic runs in
libttcross (CUDA).  The helpers ``owned_interfaces`` and ``allgather_slices`` hold the host
logic and are tested on CPU with the gloo backend (tests/test_dist_cpu.py).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .binding import TTCross


def part_begin(nif: int, world: int, p: int) -> int:
    """First interface of rank p in the balanced partition of ``nif`` interfaces."""
    q, m = divmod(nif, world)
    return p * q + min(p, m)


def owned_interfaces(d: int, rank: int, world: int):
    """[kb, ke) of the interfaces owned by ``rank`` and the exchange slot size ``chunk``
    (records per rank slot = the largest share), the rule of libttcross (part_begin)."""
    chunk = (d - 1 + world - 1) // world
    return part_begin(d - 1, world, rank), part_begin(d - 1, world, rank + 1), chunk


def record_stride(d: int, cap: int) -> int:
    """int32 per pivot record: [r, PIV[cap][d], PAR[cap][2]] (include/ttcross.h)."""
    return 1 + cap * d + 2 * cap


def pack_records(piv, par, d: int, cap: int, nrec: int):
    """Host encoding of pivot sets in the exchange-buffer layout (int32, -1 padded)."""
    rs = record_stride(d, cap)
    out = torch.full((nrec * rs,), -1, dtype=torch.int32)
    for k, (P, Q) in enumerate(zip(piv, par)):
        r = len(P)
        base = k * rs
        out[base] = r
        out[base + 1: base + 1 + r * d] = torch.as_tensor(P, dtype=torch.int32).reshape(-1)
        out[base + 1 + cap * d: base + 1 + cap * d + 2 * r] = torch.as_tensor(Q, dtype=torch.int32).reshape(-1)
    return out


def unpack_records(buf, d: int, cap: int, n_interfaces: int):
    """Inverse of pack_records: ([PIV[k] (r_k, d)], [PAR[k] (r_k, 2)]) as int64 tensors."""
    rs = record_stride(d, cap)
    buf = torch.as_tensor(buf).to(torch.int64).cpu()
    piv, par = [], []
    for k in range(n_interfaces):
        base = k * rs
        r = int(buf[base])
        piv.append(buf[base + 1: base + 1 + r * d].reshape(r, d).clone())
        par.append(buf[base + 1 + cap * d: base + 1 + cap * d + 2 * r].reshape(r, 2).clone())
    return piv, par


def pack_slots(rec, d: int, cap: int, world: int):
    """Exchange-buffer layout from interface-indexed records (host emulation of what
    tt_cross_sweep_local writes): slot p (``chunk`` records) starts with rank p's records."""
    rs = record_stride(d, cap)
    chunk = (d - 1 + world - 1) // world
    out = torch.full((world * chunk * rs,), -1, dtype=torch.int32)
    for p in range(world):
        kb, ke, _ = owned_interfaces(d, p, world)
        out[p * chunk * rs: (p * chunk + ke - kb) * rs] = rec[kb * rs: ke * rs]
    return out


def unpack_slots(xbuf, rec, d: int, cap: int, world: int):
    """Inverse of pack_slots into interface-indexed records (what tt_cross_commit does)."""
    rs = record_stride(d, cap)
    chunk = (d - 1 + world - 1) // world
    for p in range(world):
        kb, ke, _ = owned_interfaces(d, p, world)
        rec[kb * rs: ke * rs] = xbuf[p * chunk * rs: (p * chunk + ke - kb) * rs]
    return rec


def allgather_slices(buf: torch.Tensor, per_rank: int, group=None):
    """In-place all-gather: rank p's elements buf[p*per_rank:(p+1)*per_rank] are copied to
    every rank.  ``buf`` must hold world*per_rank elements (1-D)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if buf.numel() != world * per_rank:
        raise ValueError(f"buffer has {buf.numel()} elements, expected {world}*{per_rank}")
    mine = buf[rank * per_rank:(rank + 1) * per_rank].clone()
    dist.all_gather_into_tensor(buf, mine, group=group)
    return buf


def neighbour_handles(handles, rank: int, world: int):
    """(left, right) entries of the all-gathered per-rank handle list for ``rank``: the
    neighbour ranks' handles, None at the ends of the chain (tt_cross_peer_open's contract)."""
    if len(handles) != world:
        raise ValueError(f"{len(handles)} handles for world {world}")
    return (handles[rank - 1] if rank > 0 else None), (handles[rank + 1] if rank < world - 1 else None)


class DistTTCross:
    """A TT-cross problem whose interfaces are partitioned over the ranks of ``group``.

    All device work (the library's and NCCL's) is ordered on torch's current CUDA stream.

    ``peer=True`` runs the sweeps (when every rank's superblock clusters fit its device at once;
    ``self.peer`` says whether they do) as the cross-GPU wavefront (include/ttcross.h,
    tt_cross_sweep_peer): each rank's superblocks in ONE persistent launch per call, the
    boundary superblocks exchanging their new records with the neighbour ranks' kernels through
    CUDA IPC peer memory (Alg. 6 lines 6-8: neighbours only), and one all-gather of
    the records per call instead of one per sweep.  Needs a device per rank (IPC handles cannot
    be opened by their own process) with peer access between neighbours.
    """

    def __init__(self, family, u, w, rank_cap, tol, n_samples=32, rook_iters=4, seed=0, group=None,
                 fold_weights=False, peer=False):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.stream = torch.cuda.current_stream()
        self.tt = TTCross(family, u, w, rank_cap, tol, n_samples=n_samples, rook_iters=rook_iters, seed=seed,
                          rank=self.rank, world=self.world, stream=self.stream.cuda_stream, fold_weights=fold_weights)
        dev = torch.device("cuda", torch.cuda.current_device())
        xv, xper = self.tt.exchange_view()
        self.xbuf = torch.as_tensor(xv, device=dev)
        self.xper = xper // 4
        pv, pper = self.tt.partials_view()
        self.pbuf = torch.as_tensor(pv, device=dev)
        self.pper = pper // 8
        self.d = self.tt.d
        self.peer = bool(peer) and self.world > 1
        if self.peer:
            # every rank's superblocks must be resident at once (the persistent launch)
            ok = torch.tensor([1 if self.tt.launch_shape()["all_resident"] else 0], dtype=torch.int32, device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
            self.peer = bool(ok.item())
        if self.peer:
            handles = [None] * self.world
            dist.all_gather_object(handles, self.tt.peer_handles(), group=self.group)
            left, right = neighbour_handles(handles, self.rank, self.world)
            self.tt.peer_open(left, right)
            self._bar = torch.zeros(1, dtype=torch.int32, device=dev)

    def _device_barrier(self):
        """Every rank's work enqueued so far has completed on its device before anything this rank
        enqueues next runs (a one-element all-reduce on the stream): the neighbours' kernels write
        into this rank's record buffers, so no rank may start before every reset / commit is done."""
        dist.all_reduce(self._bar, group=self.group)

    def reset(self):
        self.tt.reset()
        if self.peer:
            self._device_barrier()

    def sweep(self, n_sweeps=1):
        """n_sweeps Alg. 6 sweeps: local superblock updates, all-gather of the records, commit
        (peer: one persistent launch of n_sweeps, the neighbour exchange in peer memory, then one
        all-gather + commit)."""
        if self.peer:
            if n_sweeps < 1:
                return
            self.tt.sweep_peer(n_sweeps)
            allgather_slices(self.xbuf, self.xper, self.group)
            self.tt.commit()
            self._device_barrier()
            return
        for _ in range(n_sweeps):
            self.tt.sweep_local()
            allgather_slices(self.xbuf, self.xper, self.group)
            self.tt.commit()

    def integrate_launch(self):
        self.tt.integrate_local()
        allgather_slices(self.pbuf, self.pper, self.group)

    def integrate(self):
        self.integrate_launch()
        return self.tt.integrate_finish()

    def solve(self, n_sweeps):
        """reset + n_sweeps sweeps + quadrature; returns (value, log10|value|, sign)."""
        self.reset()
        self.sweep(n_sweeps)
        return self.integrate()

    def close(self):
        self.tt.close()
