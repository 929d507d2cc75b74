"""The multi-GPU path through a real NCCL process group (one process per GPU; the pool has one
GPU, so world = 1): DistTTCross's local sweeps, exchange-slot all-gathers and commits, and the
all-gathered partial chain products give the single-context solve's pivots bit for bit and its
integral to double-double rounding."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name", ["D5", "C10"])
def test_dist_nccl_world1_equals_single(lib, name):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1", "--master-addr",
           "127.0.0.1", "--master-port", str(free_port()), os.path.join(ROOT, "tools", "dist_check.py"), name]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    assert d["world"] == 1 and d["pivots_equal"]
    assert d["rel_diff"] <= 1e-13, d


def test_bench_spawns_its_ranks(lib):
    """bench.py --gpus 1 under its own launcher logic stays single-process; the spawn path for
    --gpus N > 1 is exercised by the driver's scaling run (one GPU here)."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--workload", "C4", "--steps", "3",
                          "--warmup", "3", "--no-cpu-baseline"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert d["n_gpus"] == 1 and d["value"] > 0
