"""Thin ctypes binding of libttcross (include/ttcross.h).

Argument marshalling only: every step of the TT-cross hot path runs in the CUDA kernels of
``libttcross.so``.  There is no CPU fallback: if the shared library is missing or a call
fails, an exception is raised.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TTC_LIB_PATH") or os.path.join(HERE, "libttcross.so")   # (override: build variants)

TTC_OK = 0
TTC_FAMILY_C = 0
TTC_FAMILY_D = 1
TTC_FAMILY_CX = 2
TTC_FAMILY_DX = 3
TTC_FAMILY_EX = 4
TTC_MEM_HOST = 0
TTC_MEM_DEVICE = 1
TTC_PEER_HANDLE_BYTES = 192   # include/ttcross.h

# every symbol declared in include/ttcross.h (checked by tests/test_abi.py)
EXPORTS = [
    "tt_cross_init", "tt_cross_load_grid", "tt_cross_reset", "tt_cross_sweep", "tt_cross_sweep_local",
    "tt_cross_commit", "tt_cross_exchange_buffer", "tt_solve_launch", "tt_integrate", "tt_integrate_launch",
    "tt_integrate_read", "tt_integrate_local", "tt_integrate_partials_buffer", "tt_integrate_finish",
    "tt_cross_get_state", "tt_cross_get_fiber", "tt_cross_get_stats", "tt_cross_get_kernel_time",
    "tt_cross_set_timing", "tt_cross_destroy", "tt_last_error", "tt_build_info", "tt_cross_get_launch_shape",
    "tt_cross_get_phase_times", "tt_selftest_division", "tt_cross_get_wsum",
    "tt_cross_peer_handles", "tt_cross_peer_open", "tt_cross_sweep_peer", "tt_cross_set_loopback",
    "tt_cross_get_loopback",
]
N_KERNELS = 13


class TtcConfig(ctypes.Structure):
    _fields_ = [
        ("family", ctypes.c_int32), ("d", ctypes.c_int32), ("n", ctypes.c_int32),
        ("rank_cap", ctypes.c_int32), ("n_samples", ctypes.c_int32), ("rook_iters", ctypes.c_int32),
        ("tol", ctypes.c_double), ("seed", ctypes.c_uint64), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
        ("fold_weights", ctypes.c_int32),
    ]


class TtcStats(ctypes.Structure):
    _fields_ = [
        ("evals", ctypes.c_int64), ("launches", ctypes.c_int64), ("sweeps", ctypes.c_int32), ("pad", ctypes.c_int32),
        ("ms_fiber", ctypes.c_double), ("ms_cross", ctypes.c_double), ("ms_quad", ctypes.c_double),
        ("ms_other", ctypes.c_double), ("fiber_entries", ctypes.c_int64), ("sb_entries", ctypes.c_int64),
        ("sb_updates", ctypes.c_int64), ("rook_steps", ctypes.c_int64), ("ext_entries", ctypes.c_int64),
        ("ext_updates", ctypes.c_int64), ("ring_steps", ctypes.c_int64),
    ]


_lib = None


def load(path: str = LIB_PATH):
    """Load libttcross.so (raises FileNotFoundError / OSError if it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    P = ctypes.c_void_p
    i32, i64, f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    sig = {
        "tt_cross_init": (i32, [ctypes.POINTER(P), ctypes.POINTER(TtcConfig), P, P, i32, P]),
        "tt_cross_reset": (i32, [P]),
        "tt_cross_sweep": (i32, [P, i32]),
        "tt_cross_sweep_local": (i32, [P]),
        "tt_cross_commit": (i32, [P]),
        "tt_cross_exchange_buffer": (i32, [P, ctypes.POINTER(P), ctypes.POINTER(i64), ctypes.POINTER(i64)]),
        "tt_integrate": (i32, [P, ctypes.POINTER(f64), ctypes.POINTER(f64), ctypes.POINTER(i32)]),
        "tt_integrate_local": (i32, [P]),
        "tt_integrate_partials_buffer": (i32, [P, ctypes.POINTER(P), ctypes.POINTER(i64), ctypes.POINTER(i64)]),
        "tt_integrate_finish": (i32, [P, ctypes.POINTER(f64), ctypes.POINTER(f64), ctypes.POINTER(i32)]),
        "tt_cross_get_state": (i32, [P, P, P, P]),
        "tt_cross_get_fiber": (i32, [P, i32, P, i64, ctypes.POINTER(i32), ctypes.POINTER(i32)]),
        "tt_cross_get_stats": (i32, [P, ctypes.POINTER(TtcStats)]),
        "tt_cross_get_wsum": (i32, [P, i32, P, P, i64, ctypes.POINTER(i32), ctypes.POINTER(i32)]),
        "tt_cross_set_timing": (i32, [P, i32]),
        "tt_cross_destroy": (None, [P]),
        "tt_cross_load_grid": (i32, [P, P, P, i32]),
        "tt_cross_get_phase_times": (i32, [P, P, i32]),
        "tt_cross_get_launch_shape": (i32, [P, ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(i32),
                                            ctypes.POINTER(i64)]),
        "tt_cross_get_kernel_time": (i32, [P, i32, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(i64),
                                           ctypes.POINTER(f64)]),
        "tt_solve_launch": (i32, [P, i32, i32]),
        "tt_integrate_launch": (i32, [P]),
        "tt_integrate_read": (i32, [P, ctypes.POINTER(f64), ctypes.POINTER(f64), ctypes.POINTER(i32)]),
        "tt_last_error": (ctypes.c_char_p, []),
        "tt_build_info": (ctypes.c_char_p, []),
        "tt_selftest_division": (i32, [P, P, P, P, i64]),
        "tt_cross_peer_handles": (i32, [P, P, i64]),
        "tt_cross_peer_open": (i32, [P, P, P]),
        "tt_cross_sweep_peer": (i32, [P, i32]),
        "tt_cross_set_loopback": (i32, [P, i32]),
        "tt_cross_get_loopback": (i32, [P, P, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name, None)
        if fn is None and os.environ.get("TTC_LIB_PATH"):
            continue   # (an older build variant for A/B runs; tests/test_abi.py checks the product library)
        if fn is None:
            raise OSError(f"{path}: symbol {name} missing (stale build?)")
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class TTCError(RuntimeError):
    pass


def _check(lib, rc, what):
    if rc != TTC_OK:
        raise TTCError(f"{what} failed (code {rc}): {lib.tt_last_error().decode()}")


def _ptr_and_kind(arr):
    """(pointer, mem_kind, keepalive) for a numpy array or a CUDA tensor/array."""
    if hasattr(arr, "__cuda_array_interface__") and not isinstance(arr, np.ndarray):
        iface = arr.__cuda_array_interface__
        if iface["typestr"] != "<f8":
            raise TypeError("device arrays must be float64")
        return ctypes.c_void_p(iface["data"][0]), TTC_MEM_DEVICE, arr
    a = np.ascontiguousarray(arr, dtype=np.float64)
    return a.ctypes.data_as(ctypes.c_void_p), TTC_MEM_HOST, a


class DeviceView:
    """__cuda_array_interface__ wrapper of a library-owned device buffer (zero copy)."""

    def __init__(self, ptr, nbytes, typestr):
        self.ptr, self.nbytes, self.typestr = ptr, nbytes, typestr
        itemsize = int(typestr[2:])
        self.__cuda_array_interface__ = {
            "shape": (nbytes // itemsize,), "typestr": typestr, "data": (ptr, False), "version": 2,
        }


class TTCross:
    """Handle on one TT-cross problem (C-ABI context)."""

    def __init__(self, family, u, w, rank_cap, tol, n_samples=32, rook_iters=4, seed=0, rank=0, world=1,
                 stream=None, fold_weights=False):
        self.lib = load()
        self.d, self.n = int(u.shape[0]), int(u.shape[1])
        self.cap = int(rank_cap)
        self.cfg = TtcConfig(int(family), self.d, self.n, self.cap, int(n_samples), int(rook_iters), float(tol),
                             int(seed) & ((1 << 64) - 1), int(rank), int(world), 1 if fold_weights else 0)
        pu, ku, keep_u = _ptr_and_kind(u)
        pw, kw, keep_w = _ptr_and_kind(w)
        if ku != kw:
            raise TypeError("nodes and weights must both be host or both be device arrays")
        self._h = ctypes.c_void_p()
        # the library copies the grid asynchronously on its stream: the source buffers stay
        # referenced here until a synchronising call (include/ttcross.h, tt_cross_init)
        self._inflight = [keep_u, keep_w]
        sp = ctypes.c_void_p(int(stream)) if stream else ctypes.c_void_p()
        _check(self.lib, self.lib.tt_cross_init(ctypes.byref(self._h), ctypes.byref(self.cfg), pu, pw, ku, sp),
               "tt_cross_init")

    # -- lifecycle
    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self.lib.tt_cross_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reset(self):
        _check(self.lib, self.lib.tt_cross_reset(self._h), "tt_cross_reset")

    def set_timing(self, on=True):
        _check(self.lib, self.lib.tt_cross_set_timing(self._h, 1 if on else 0), "tt_cross_set_timing")

    # -- the hot path
    def sweep(self, n_sweeps=1):
        _check(self.lib, self.lib.tt_cross_sweep(self._h, int(n_sweeps)), "tt_cross_sweep")

    def sweep_local(self):
        _check(self.lib, self.lib.tt_cross_sweep_local(self._h), "tt_cross_sweep_local")

    def commit(self):
        _check(self.lib, self.lib.tt_cross_commit(self._h), "tt_cross_commit")

    def integrate(self):
        v, l10, sg = ctypes.c_double(), ctypes.c_double(), ctypes.c_int32()
        _check(self.lib, self.lib.tt_integrate(self._h, ctypes.byref(v), ctypes.byref(l10), ctypes.byref(sg)),
               "tt_integrate")
        self._synced()
        return v.value, l10.value, sg.value

    def load_grid(self, u, w):
        pu, ku, keep_u = _ptr_and_kind(u)
        pw, kw, keep_w = _ptr_and_kind(w)
        if ku != kw:
            raise TypeError("nodes and weights must both be host or both be device arrays")
        self._inflight += [keep_u, keep_w]
        _check(self.lib, self.lib.tt_cross_load_grid(self._h, pu, pw, ku), "tt_cross_load_grid")

    def _synced(self):
        """The library's stream has completed everything enqueued so far."""
        self._inflight = []

    def solve_launch(self, n_sweeps, graph=True):
        _check(self.lib, self.lib.tt_solve_launch(self._h, int(n_sweeps), 1 if graph else 0), "tt_solve_launch")

    def integrate_launch(self):
        _check(self.lib, self.lib.tt_integrate_launch(self._h), "tt_integrate_launch")

    def integrate_read(self):
        v, l10, sg = ctypes.c_double(), ctypes.c_double(), ctypes.c_int32()
        _check(self.lib, self.lib.tt_integrate_read(self._h, ctypes.byref(v), ctypes.byref(l10), ctypes.byref(sg)),
               "tt_integrate_read")
        self._synced()
        return v.value, l10.value, sg.value

    def integrate_local(self):
        _check(self.lib, self.lib.tt_integrate_local(self._h), "tt_integrate_local")

    def integrate_finish(self):
        v, l10, sg = ctypes.c_double(), ctypes.c_double(), ctypes.c_int32()
        _check(self.lib, self.lib.tt_integrate_finish(self._h, ctypes.byref(v), ctypes.byref(l10), ctypes.byref(sg)),
               "tt_integrate_finish")
        self._synced()
        return v.value, l10.value, sg.value

    # -- cross-GPU wavefront (include/ttcross.h: tt_cross_peer_handles ... tt_cross_get_loopback)
    def peer_handles(self):
        """This context's CUDA IPC handles (bytes, TTC_PEER_HANDLE_BYTES) for its neighbour ranks."""
        buf = ctypes.create_string_buffer(TTC_PEER_HANDLE_BYTES)
        _check(self.lib, self.lib.tt_cross_peer_handles(self._h, buf, TTC_PEER_HANDLE_BYTES), "tt_cross_peer_handles")
        return buf.raw

    def peer_open(self, left, right):
        """Map the neighbour ranks' handles (bytes or None)."""
        lb = ctypes.create_string_buffer(bytes(left), TTC_PEER_HANDLE_BYTES) if left is not None else None
        rb = ctypes.create_string_buffer(bytes(right), TTC_PEER_HANDLE_BYTES) if right is not None else None
        _check(self.lib, self.lib.tt_cross_peer_open(self._h, lb, rb), "tt_cross_peer_open")
        self._synced()

    def sweep_peer(self, n_sweeps):
        _check(self.lib, self.lib.tt_cross_sweep_peer(self._h, int(n_sweeps)), "tt_cross_sweep_peer")

    def set_loopback(self, boundary):
        _check(self.lib, self.lib.tt_cross_set_loopback(self._h, int(boundary)), "tt_cross_set_loopback")

    def loopback(self):
        """(records [d-1][RS] int32, rank ring [d-1][2], done [d-1]) of the loopback mirror."""
        rs = 1 + self.cap * self.d + 2 * self.cap
        rec = np.zeros((self.d - 1, rs), dtype=np.int32)
        ring = np.zeros((self.d - 1, 2), dtype=np.int32)
        done = np.zeros(self.d - 1, dtype=np.int32)
        _check(self.lib, self.lib.tt_cross_get_loopback(self._h, rec.ctypes.data_as(ctypes.c_void_p),
                                                        ring.ctypes.data_as(ctypes.c_void_p),
                                                        done.ctypes.data_as(ctypes.c_void_p)), "tt_cross_get_loopback")
        self._synced()
        return rec, ring, done

    # -- buffers for the multi-process exchange (zero-copy device views)
    def exchange_view(self):
        p, tot, per = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_int64()
        _check(self.lib, self.lib.tt_cross_exchange_buffer(self._h, ctypes.byref(p), ctypes.byref(tot),
                                                           ctypes.byref(per)), "tt_cross_exchange_buffer")
        return DeviceView(p.value, tot.value, "<i4"), per.value

    def partials_view(self):
        p, tot, per = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_int64()
        _check(self.lib, self.lib.tt_integrate_partials_buffer(self._h, ctypes.byref(p), ctypes.byref(tot),
                                                               ctypes.byref(per)), "tt_integrate_partials_buffer")
        return DeviceView(p.value, tot.value, "<f8"), per.value

    # -- inspection
    def state(self, parents=False):
        """(ranks, [PIV[k] (r_k, d)]) and, with parents=True, also [PAR[k] (r_k, 2)]."""
        ranks = np.zeros(self.d - 1, dtype=np.int32)
        piv = np.zeros((self.d - 1, self.cap, self.d), dtype=np.int32)
        par = np.zeros((self.d - 1, self.cap, 2), dtype=np.int32)
        _check(self.lib, self.lib.tt_cross_get_state(self._h, ranks.ctypes.data_as(ctypes.c_void_p),
                                                     piv.ctypes.data_as(ctypes.c_void_p),
                                                     par.ctypes.data_as(ctypes.c_void_p)), "tt_cross_get_state")
        self._synced()
        P = [piv[i, :ranks[i]].astype(np.int64) for i in range(self.d - 1)]
        if parents:
            return ranks, P, [par[i, :ranks[i]].astype(np.int64) for i in range(self.d - 1)]
        return ranks, P

    def fiber(self, mode):
        rx, ry = ctypes.c_int32(), ctypes.c_int32()
        _check(self.lib, self.lib.tt_cross_get_fiber(self._h, int(mode), None, 0, ctypes.byref(rx), ctypes.byref(ry)),
               "tt_cross_get_fiber")
        out = np.empty((rx.value, ry.value, self.n), dtype=np.float64)
        _check(self.lib, self.lib.tt_cross_get_fiber(self._h, int(mode), out.ctypes.data_as(ctypes.c_void_p),
                                                     out.size, ctypes.byref(rx), ctypes.byref(ry)),
               "tt_cross_get_fiber")
        return out

    def wsum(self, mode):
        """W_m = sum_a w_{m,a} F_m[:, :, a] in double-double as (hi, lo), each (r_{m-1}, r_m), as the
        last quadrature (or fiber()) computed it."""
        rx, ry = ctypes.c_int32(), ctypes.c_int32()
        _check(self.lib, self.lib.tt_cross_get_wsum(self._h, int(mode), None, None, 0, ctypes.byref(rx),
                                                    ctypes.byref(ry)), "tt_cross_get_wsum")
        hi = np.empty((rx.value, ry.value))
        lo = np.empty((rx.value, ry.value))
        _check(self.lib, self.lib.tt_cross_get_wsum(self._h, int(mode), hi.ctypes.data_as(ctypes.c_void_p),
                                                    lo.ctypes.data_as(ctypes.c_void_p), hi.size, ctypes.byref(rx),
                                                    ctypes.byref(ry)), "tt_cross_get_wsum")
        self._synced()
        return hi, lo

    def stats(self):
        s = TtcStats()
        _check(self.lib, self.lib.tt_cross_get_stats(self._h, ctypes.byref(s)), "tt_cross_get_stats")
        self._synced()
        return {f: getattr(s, f) for f, _ in TtcStats._fields_ if f != "pad"}


    def phase_times(self, per_sweep=False):
        """k_sweep phase clocks (us, CTA 0 of superblock TTC_PHASE_JOB, default the first) accumulated
        while timing is on; per_sweep=True also returns the per-sweep log (a list of dicts)."""
        nw = 14 + 16 * 256
        out = np.zeros(nw)
        _check(self.lib, self.lib.tt_cross_get_phase_times(self._h, out.ctypes.data_as(ctypes.c_void_p), nw),
               "tt_cross_get_phase_times")
        names = ["prologue", "tables", "extend", "samples", "rook", "final", "exit", "launches",
                 "col_eval", "col_argmax", "row_eval", "row_argmax", "ext_raw", "ext_rec"]
        tot = dict(zip(names, out[:14].tolist()))
        if not per_sweep:
            return tot
        log = out[14:].reshape(256, 16)
        rows = [dict(zip(names[:7] + ["rounds"] + names[8:] + ["ext_rows_cta", "ext_cols_cta"],
                         [round(x, 2) for x in r.tolist()])) for r in log]
        while rows and not any(rows[-1].values()):
            rows.pop()
        return tot, rows

    def launch_shape(self):
        g, t, ca, sm = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64()
        _check(self.lib, self.lib.tt_cross_get_launch_shape(self._h, ctypes.byref(g), ctypes.byref(t), ctypes.byref(ca),
                                                            ctypes.byref(sm)), "tt_cross_get_launch_shape")
        return {"cluster": g.value, "threads": t.value, "cached": bool(ca.value & 1), "persistent": bool(ca.value & 2),
                "all_resident": bool(ca.value & 4),
                "smem_bytes": sm.value}

    def kernel_times(self):
        """{kernel name: (launches, ms)} since the last reset (ms only with timing on)."""
        out = {}
        for k in range(N_KERNELS):
            nm, nl, ms = ctypes.c_char_p(), ctypes.c_int64(), ctypes.c_double()
            _check(self.lib, self.lib.tt_cross_get_kernel_time(self._h, k, ctypes.byref(nm), ctypes.byref(nl),
                                                               ctypes.byref(ms)), "tt_cross_get_kernel_time")
            out[nm.value.decode()] = (nl.value, ms.value)
        return out


def build_info():
    return load().tt_build_info().decode()
