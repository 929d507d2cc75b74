#!/usr/bin/env python
"""bench.py -- throughput of the B200 TT-cross quadrature hot path (arXiv:1903.11554).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload D5] [--impl ours|reference]

A *step* is one whole solve of the workload: reset to the seed-fixed rank-1
start, the workload's dimension-parallel sweeps (Alg. 6: every superblock, at
once, extends its cross to the new rows/columns -- the batched fiber evaluation -- and adds
one pivot found by Alg. 2) and the TT quadrature (§4.1).  ``value`` = integrand evaluations per second (the device
counter of evaluated tensor entries ÷ device time), whole job, inputs resident in HBM.

N = 1: the solve is one CUDA graph replayed per step (tt_solve_launch).  N > 1 (torchrun,
one process per GPU, NCCL): interfaces are partitioned over ranks and the new pivots are
all-gathered after every half-sweep (paper_1903_11554_b200.dist); total work is fixed, so
scaling is "strong".  Timing: CUDA events on the library's stream around each step, L2
flushed (256 MiB memset) before every timed step, barrier + synchronize on both sides, max
over ranks.  ``e2e`` runs the same steps through the public API from pinned host buffers:
tt_cross_load_grid (H2D of nodes + weights) -> tt_solve_launch -> tt_integrate_read (D2H of
the result), timed by the host clock.  ``roofline`` comes from a second pass of the same
steps with per-kernel CUDA events enabled (tt_cross_set_timing), for the kernel with the
largest device time.  ``cpu_baseline`` times the oracle (test infrastructure, never the
product path) on a bounded sample on rank 0.

--impl reference: the oracle as the reference arm: each step is a bounded
sample of the same workload on the host cores, same metric and unit.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from workloads import FAMILY_NAMES, WORKLOADS, X_FAMILIES, X_WORKLOADS  # noqa: E402

ALL_WORKLOADS = {**WORKLOADS, **X_WORKLOADS}

DEFAULT_WORKLOAD = "D20"   # BASELINE.json configs[3]: the largest single-GPU config
L2_FLUSH_BYTES = 256 << 20
# fp64 peak: MEASURED on this pool's B200 by tools/fp64_peak.cu (DFMA chains
# on every SM, CUDA events; profiles/fp64_peak.json), else the nominal 148 SMs x 64 FP64 FMA
# lanes x 2 flop x 1.965 GHz
FP64_NOMINAL_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12


def fp64_peak(mode="burst"):
    """(TFLOP/s, source): the measured DFMA throughput ('burst': a kernel timed alone;
    'sustained': back to back for seconds), or the nominal figure."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            e = json.load(f)
        return float(e[f"dfma_{mode}_tflops"]), f"measured DFMA {mode} (profiles/fp64_peak.json, tools/fp64_peak.cu)"
    except Exception:
        return FP64_NOMINAL_TFLOPS, "nominal: 148 SM x 64 FP64 lanes x 2 flop x 1.965 GHz (no measurement committed)"


FP64_PEAK_TFLOPS, FP64_PEAK_SOURCE = fp64_peak()


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(ALL_WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of the CUDA graph")
    ap.add_argument("--no-peer", action="store_true",
                    help="N > 1: one launch + NCCL all-gather per sweep instead of the cross-GPU wavefront")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="budget of the oracle sample")
    return ap.parse_args()


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


# --------------------------------------------------------------------------------------
# clocks during the timed region
# --------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                p = [x.strip() for x in line.split(",")]
                if len(p) >= 9:
                    rows.append(p)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# --------------------------------------------------------------------------------------
# roofline of the dominant kernel
# --------------------------------------------------------------------------------------
# algorithmic fp64 flops per superblock entry: C: S = H + L*2^-52 (2), S*S (1),
# 1/S^2 (1); D: + five double-double products (10 each), rho (4), dd * rho (8), rounding and
# the division (2).  x-form (m modes): prefix/suffix products and sums 4m, B 2; each of the
# m(m+1)/2 pairs 6 (running product, 1-p, 1+p, division, q*q, accumulate).
def flops_per_entry(family, m):
    if family == 0:
        return 4
    if family == 1:
        return 68
    pairs = 3 * m * (m + 1)
    return {2: 4 * m + 2, 3: 4 * m + 3 + pairs, 4: pairs}[family]


# algorithmic fp64 flops per entry of the fused quadrature fiber kernel, an
# FMA counted as 2 and an IEEE division or reciprocal as 1:  rounding of the exact sum S (2),
# S*S (1);  D only: two double-double products (10 each: p, err FMA, two FMAs, s, l), hi+lo
# (1), the division (1);  C: the reciprocal (1);  the double-double accumulation of w_a*A
# (14: product + error FMA, two-sum, renormalisation).  C 18, D 39.  (ncu's executed fp64
# operations are higher -- C 27.2, D 53.3 per entry, profiles/r01n_ncu_fiber_wsum_*_flops.csv
# -- because the IEEE division expands into a reciprocal and Newton steps.)
FIBER_FLOPS_PER_ENTRY = {0: 18, 1: 39}


def fiber_roofline(kt, stats, family, modes, peaks):
    """The quadrature fiber kernel: the throughput-mode batched integrand evaluation.
    t-form (k_fiber_wsum, fused with the weighted sum, nothing written per entry):
    FIBER_FLOPS_PER_ENTRY; x-form (k_fiber_x, 8 B written per entry): flops_per_entry."""
    launches, ms = kt.get("k_fiber", (0, 0.0))
    if not launches or ms <= 0:
        return None
    avg_s = ms / launches / 1e3
    ent = stats["fiber_entries"] / launches
    fused = family in (0, 1)
    fpe = FIBER_FLOPS_PER_ENTRY[family] if fused else flops_per_entry(family, modes)
    tf = ent * fpe / avg_s / 1e12
    gbs = 0.0 if fused else ent * 8 / avg_s / 1e9
    return {"kernel": "k_fiber_wsum" if fused else "k_fiber_x", "avg_us": avg_s * 1e6, "entries_per_launch": ent,
            "achieved_tflops": tf, "frac_fp64_peak": tf / FP64_PEAK_TFLOPS, "fp64_peak_tflops": FP64_PEAK_TFLOPS,
            "fp64_peak_source": FP64_PEAK_SOURCE,
            "write_GBs": gbs, "frac_hbm": gbs / peaks["hbm_gbs"],
            "per_unit": f"{fpe} flop / entry" + ("" if fused else " + 8 B written")}


def ncu_traffic(workload, kernel):
    """DRAM bytes per launch of the dominant kernel from the committed `ncu --set full`
    capture (profiles/ncu_traffic.json, written by tools/ncu_report.py), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            e = json.load(f).get(workload)
    except Exception:
        return None, None
    if not e or not e["kernel"].startswith(kernel):
        return None, None
    return e["dram_bytes_per_launch"], e["source"]


def roofline(kt, stats, family, peaks, peak_src, modes=0, workload=None, cached=False):
    """kt: {name: (launches, ms)} of the profiling pass; stats: its summed counters.
    The bound is the roof the kernel's algorithmic work comes closest to: fp64 flops against
    the derived fp64 peak, or -- when the rook steps stream the u/v factors from memory (not
    the cached launch shape) -- algorithmic bytes against the measured HBM bandwidth."""
    name = max(kt, key=lambda k: kt[k][1])
    launches, ms = kt[name]
    avg_s = ms / max(1, launches) / 1e3
    traffic, tsrc = ncu_traffic(workload, name + "s" if name == "k_sweep" else name)
    out = {"kernel": name, "avg_us": avg_s * 1e6, "launches": launches, "traffic": traffic}
    if traffic is not None:
        out["traffic_source"] = tsrc
    fpe = flops_per_entry(family, modes)
    if name == "k_sweep":
        ent = stats["sb_entries"] / max(1, launches)
        upd = stats["sb_updates"] / max(1, launches)
        out["rook_steps_per_launch"] = stats["rook_steps"] / max(1, launches)
        out["extension_share_of_entries"] = stats["ext_entries"] / max(1, stats["sb_entries"])
    elif name == "k_fiber":
        ent, upd = stats["fiber_entries"] / max(1, launches), 0
    else:
        out.update({"bound": "latency", "achieved": None, "peak": None, "unit": None, "frac": None,
                    "peak_source": None})
        return out
    flops = ent * fpe + 2 * upd   # one multiply + one subtract per u_t(x) v_t(y) term
    tf = flops / avg_s / 1e12
    alu = {"bound": "alu", "achieved": tf, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
           "frac": tf / FP64_PEAK_TFLOPS,
           "per_unit": f"{fpe} fp64 flop/entry + 2 flop/update term",
           "peak_source": FP64_PEAK_SOURCE}
    out.update({"entries_per_launch": ent, "updates_per_launch": upd})
    if name == "k_sweep" and not cached:
        # memory side: in the samples and rook steps every u_t(x) v_t(y) term
        # streams one factor from HBM (the other is staged) and every entry writes its E and raw
        # value (16 B); the u/v extension works on chip and writes one 8-byte u/v value per entry
        # value (16 B) and reads its row's (column's) own-side factor tables: SA (16 B) for the
        # C family, SA + PA (16 + 24 B) for D -- per row and step, too many to stay on chip in
        # the streaming shapes
        ext_e = stats["ext_entries"] / max(1, launches)
        ext_u = stats["ext_updates"] / max(1, launches)
        tab = 40 if family == 1 else (16 if family == 0 else 0)
        algo = 8 * (upd - ext_u) + (16 + tab) * (ent - ext_e) + 8 * ext_e
        gbs = algo / avg_s / 1e9
        hbm = {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
               "frac": gbs / peaks["hbm_gbs"], "bytes_per_launch": algo,
               "per_unit": f"8 B/streamed update term + {16 + tab} B/search entry (E and raw written, "
                           f"{tab} B of own-side tables read) + 8 B/extension entry",
               "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})"}
        main, other = (hbm, alu) if hbm["frac"] >= alu["frac"] else (alu, hbm)
        out.update(main)
        out["other_roof"] = other
    else:
        out.update(alu)
    out["limiter"] = ("latency: the dependent argmax chain of Alg. 2 (DESIGN.md 5b)" if name == "k_sweep"
                      and out["frac"] < 0.1 else "throughput")
    return out


# --------------------------------------------------------------------------------------
# oracle leg (cpu_baseline and --impl reference)
# --------------------------------------------------------------------------------------
_ORACLE_PROB = None


def _oracle_init(name):
    global _ORACLE_PROB
    from oracle import cross as X
    wl = ALL_WORKLOADS[name]
    u, w = wl.grid()
    _ORACLE_PROB = X.Problem(wl.family, u, w, wl.rank_cap, wl.tol, wl.n_samples, wl.rook_iters, wl.seed, wl.fold)


def _oracle_solve(nsw):
    from oracle import cross as X
    st, val, _ = X.run(_ORACLE_PROB, nsw)
    return st.n_evals


def _oracle_update(args):
    from oracle import cross as X
    st, k = args
    piv, par, info = X.superblock_update(_ORACLE_PROB, st, k)
    return k, piv, par, info["evals"]


def oracle_pool(wl, cores=None):
    """A process pool for oracle_sample (numpy single-threaded in every process)."""
    import multiprocessing as mp
    cores = cores or os.cpu_count() or 1
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"
    return mp.get_context("fork").Pool(cores, initializer=_oracle_init, initargs=(wl.name,)), cores


def oracle_sample(wl, budget_s, cores=None, pool=None):
    """Run the oracle (test infrastructure, as it stands) on a bounded sample of the workload
    on `cores` host processes (numpy, one thread each); returns (evals, seconds, what, cores,
    solve_s or None).

    Small workloads (a whole solve takes ~1 s on one core): whole solves, one per process,
    repeated while the budget lasts.  Large ones: Alg. 6 sweeps from the rank-1 start, the
    superblock updates of a sweep spread over the processes (each = LU of the existing
    cross + one Alg. 2 step, Alg. 6), stopped after the sweep in
    which the budget runs out.
    """
    from oracle import cross as X
    _oracle_init(wl.name)
    prob = _ORACLE_PROB
    nsw = wl.alg6_sweeps
    own = pool is None
    if own:
        pool, cores = oracle_pool(wl, cores)
    else:
        cores = cores or os.cpu_count() or 1
    evals = 0
    try:
        if True:
            t0 = time.perf_counter()
            if wl.d <= 8:
                solves = 0
                while True:
                    for e in pool.imap_unordered(_oracle_solve, [nsw] * cores):
                        evals += e
                        solves += 1
                    if time.perf_counter() - t0 > budget_s:
                        break
                s = time.perf_counter() - t0
                return (evals, s, f"{solves} full solve(s) ({nsw} Alg. 6 sweeps + quadrature), {cores} at a time",
                        cores, s / solves * cores)
            st = X.initial_state(prob)
            sweeps = 0
            while time.perf_counter() - t0 <= budget_s and sweeps < nsw:
                new = st.copy()
                for k, piv, par, ev in pool.imap_unordered(_oracle_update, [(st, k) for k in range(wl.d - 1)]):
                    new.piv[k], new.par[k] = piv, par
                    evals += ev
                new.sweep = st.sweep + 1
                st = new
                sweeps += 1
            return (evals, time.perf_counter() - t0,
                    f"the first {sweeps} Alg. 6 sweeps from the rank-1 start (ranks up to {max(st.ranks)}), "
                    f"superblocks spread over {cores} processes", cores, None)
    finally:
        if own:
            pool.close()
            pool.join()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl = ALL_WORKLOADS[args.workload]
    budget = max(0.5, min(args.cpu_seconds, 150.0 / max(1, args.steps + args.warmup)))
    pool, cores = oracle_pool(wl)   # (one pool for the run: the workers start once)
    for _ in range(args.warmup):
        oracle_sample(wl, budget, cores, pool)
    tot_e, tot_s, what = 0, 0.0, ""
    for _ in range(args.steps):
        e, s, what, cores, _ = oracle_sample(wl, budget, cores, pool)
        tot_e += e
        tot_s += s
    pool.close()
    pool.join()
    v = tot_e / tot_s
    line = {
        "impl": "reference", "metric": "integrand evals/sec (fp64)", "value": v, "unit": "evals/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_s / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(wl, args.gpus),
        "cpu_baseline": {"value": v, "unit": "evals/s", "cores": cores, "kind": "oracle",
                         "sample": f"per step: {what} of {wl.name} (numpy fp64, one thread per process)"},
        "e2e": {"value": v, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(wl, n):
    return {"workload": f"{FAMILY_NAMES[wl.family]}_{wl.d}", "d": wl.d, "modes": wl.modes, "n": wl.n,
            "rule": "gauss-legendre [0,1]" if wl.family in X_FAMILIES else f"trapezoid [-{wl.L:g},{wl.L:g}]",
            "rank_cap": wl.rank_cap, "tol": wl.tol, "sweeps": wl.sweeps, "alg6_sweeps": wl.alg6_sweeps,
            "n_samples": wl.n_samples, "rook_iters": wl.rook_iters, "seed": wl.seed,
            "parallelism": f"superblocks/{n}",
            "fold_weights": wl.fold, "l2": "flushed (256 MiB memset) before every timed step"}


# --------------------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------------------
def spawn_ranks(args):
    """--gpus N > 1 without a launcher: start N ranks (one process per GPU) through
    torch.distributed.run on 127.0.0.1 and pass their output through."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def nccl_summary(path_glob):
    """One stderr line from the NCCL_DEBUG=INFO logs of this job: communicator ranks, channels,
    whether NVLS (in-switch reduction) was set up."""
    import glob
    lines = []
    for p in glob.glob(path_glob):
        with open(p, errors="replace") as f:
            lines += f.readlines()
    nvls = any("NVLS" in ln for ln in lines)
    ranks = sorted({ln.split("rank ")[1].split()[0] for ln in lines if "Init COMPLETE" in ln and "rank " in ln})
    chans = sum(1 for ln in lines if "via P2P" in ln or "via NVLS" in ln)
    print(f"[bench] NCCL: {len(lines)} log lines, comm ranks {ranks}, {chans} P2P/NVLS channel lines, "
          f"NVLS {'seen' if nvls else 'not seen'} ({path_glob})", file=sys.stderr, flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(spawn_ranks(args))
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    nccl_log = None
    if world > 1:
        # communicator ranks / channels / NVLS visible without polluting stdout (the JSON line)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        nccl_log = os.path.join(tempfile.gettempdir(), f"ttc_nccl_{os.environ.get('MASTER_PORT', '0')}")
        os.environ.setdefault("NCCL_DEBUG_FILE", nccl_log + ".%h.%p.log")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_1903_11554_b200 import TTCross
    from paper_1903_11554_b200.dist import DistTTCross

    wl = ALL_WORKLOADS[args.workload]
    u, w = wl.grid()
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    u_d = torch.from_numpy(u).to(dev)
    w_d = torch.from_numpy(w).to(dev)
    kw = dict(n_samples=wl.n_samples, rook_iters=wl.rook_iters, seed=wl.seed)
    if wl.fold:
        kw["fold_weights"] = True
    nsw = wl.alg6_sweeps
    use_graph = world == 1 and not args.no_graph
    if world == 1:
        tt = TTCross(wl.family, u_d, w_d, wl.rank_cap, wl.tol, stream=stream.cuda_stream, **kw)

        def step():
            tt.solve_launch(nsw, graph=use_graph)

        def result():
            return tt.integrate_read()
        core = tt
    else:
        dtt = DistTTCross(wl.family, u_d, w_d, wl.rank_cap, wl.tol, peer=not args.no_peer, **kw)

        last = {}

        def step():
            last["v"] = dtt.solve(nsw)

        def result():
            return last["v"]
        core = dtt.tt

    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    t_ramp = time.perf_counter()
    while time.perf_counter() - t_ramp < 0.3:  # let the SM clock leave idle before warm-up
        flush.zero_()
        torch.cuda.synchronize()
    for _ in range(max(3, args.warmup)):
        step()
        val = result()
    barrier()
    st0 = core.stats()
    evals_step = st0["evals"]
    launches_step = st0["launches"]

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    for k in range(args.steps):
        flush.zero_()
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
    barrier()
    clocks = sampler.stop()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    val = result()
    t = torch.tensor([ms, float(evals_step)], dtype=torch.float64, device=dev)
    if world > 1:
        tmax = t[:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t[1:].clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        ms_max, evals_total = float(tmax.item()), float(tsum.item())
    else:
        ms_max, evals_total = ms, float(evals_step)
    value = evals_total * args.steps / (ms_max / 1e3)

    # ---- end to end through the public API from pinned host buffers (host clock)
    u_h = torch.from_numpy(u).pin_memory()
    w_h = torch.from_numpy(w).pin_memory()
    h2d = 2 * u.size * 8
    d2h = 2 * 8 + 4
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        core.load_grid(u_h.numpy(), w_h.numpy())
        if world == 1:
            tt.solve_launch(nsw, graph=use_graph)
            e2e_val = tt.integrate_read()
        else:
            dtt.sweep(nsw)
            e2e_val = dtt.integrate()
    barrier()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_s = float(te.item())
    e2e = {"value": evals_total * args.steps / e2e_s, "unit": "evals/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "timer": "host clock around synchronous steps"}

    # ---- per-kernel profile pass (eager launches, CUDA events around every launch); every
    # solve resets the library's counters, so they are accumulated here solve by solve
    nprof = max(3, min(args.steps, 50))
    barrier()
    core.set_timing(True)
    kt, st = {}, {}
    for _ in range(nprof):
        if world == 1:
            tt.solve_launch(nsw, graph=False)
            tt.integrate_read()
        else:
            dtt.solve(nsw)
        for k, (nl, kms) in core.kernel_times().items():
            a, b = kt.get(k, (0, 0.0))
            kt[k] = (a + nl, b + kms)
        for k, v in core.stats().items():
            st[k] = st.get(k, 0) + v
    core.set_timing(False)
    peaks, peak_src = measured_peaks()
    roof = roofline(kt, st, wl.family, peaks, peak_src, wl.modes, workload_config(wl, world)["workload"],
                    core.launch_shape()["cached"])
    froof = fiber_roofline(kt, st, wl.family, wl.modes, peaks)
    kernel_ms = {k: v[1] / nprof for k, v in kt.items() if v[0]}

    # ---- oracle on the host cores (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        e, s, what, cores, solve_s = oracle_sample(wl, args.cpu_seconds)
        cpu = {"value": e / s, "unit": "evals/s", "cores": cores, "kind": "oracle",
               "sample": f"{what} of {wl.name} (numpy fp64, one thread per process), {s:.1f} s",
               "solve_s_per_core": solve_s}

    if rank == 0:
        line = {
            "metric": "integrand evals/sec (fp64)", "value": value, "unit": "evals/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(wl, world),
            "evals_per_step": evals_total, "sweep_ms": ms_max / args.steps,
            "integral": {"value": val[0], "log10_abs": val[1], "sign": val[2]},
            "graph": use_graph, "gpu_launches": int(launches_step) * args.steps,
            "exchange": ("none (one GPU)" if world == 1 else
                         "cross-GPU wavefront: boundary records through CUDA IPC peer memory, one NCCL all-gather per solve"
                         if dtt.peer else "NCCL all-gather of the new records after every sweep"),
            "launch_shape": core.launch_shape(),
            "roofline": roof, "fiber_roofline": froof, "kernel_ms_per_solve": kernel_ms, "clocks": clocks, "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
        if rank == 0 and nccl_log:
            nccl_summary(nccl_log + ".*.log")
    core.close()


if __name__ == "__main__":
    main()
