#!/usr/bin/env python
"""One process per GPU under torch.distributed.run (NCCL): DistTTCross (the multi-GPU path of
paper_1903_11554_b200.dist -- local sweeps, all-gather of the exchange slots, commit, partial
chain products) against the single-context solve of the same workload.  Rank 0 prints one JSON
line.  Used by tests/test_gpu_dist.py at world = 1 (the pool has one GPU).
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/dist_check.py D5
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "D5"
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1903_11554_b200 import TTCross
    from paper_1903_11554_b200.dist import DistTTCross, owned_interfaces
    from workloads import WORKLOADS
    wl = WORKLOADS[name]
    u, w = wl.grid()
    dev = torch.device("cuda", local)
    kw = dict(n_samples=wl.n_samples, rook_iters=wl.rook_iters, seed=wl.seed)
    dtt = DistTTCross(wl.family, torch.from_numpy(u).to(dev), torch.from_numpy(w).to(dev), wl.rank_cap, wl.tol, **kw)
    val = dtt.solve(wl.alg6_sweeps)
    ranks, piv, par = dtt.tt.state(parents=True)
    ref = TTCross(wl.family, u, w, wl.rank_cap, wl.tol, **kw)
    ref.sweep(wl.alg6_sweeps)
    rval = ref.integrate()
    rranks, rpiv, rpar = ref.state(parents=True)
    same = list(ranks) == list(rranks) and all(np.array_equal(a, b) for a, b in zip(piv + par, rpiv + rpar))
    if dist.get_rank() == 0:
        print(json.dumps({"workload": name, "world": dist.get_world_size(),
                          "partition": [owned_interfaces(wl.d, p, dist.get_world_size())[:2]
                                        for p in range(dist.get_world_size())],
                          "pivots_equal": bool(same), "integral": val[0], "integral_single": rval[0],
                          "rel_diff": abs(val[0] - rval[0]) / abs(rval[0])}), flush=True)
    dtt.close()
    ref.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
