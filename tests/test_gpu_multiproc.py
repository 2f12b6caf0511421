"""The N>1 path of bench.py end to end — torchrun, one process per rank,
patch-row shards, halo ring and metric reductions through torch.distributed
— run with 2 ranks on the ONE GPU of this box over gloo (host-staged
exchange; WG_DIST_BACKEND/WG_FORCE_DEVICE).  It checks the orchestration,
not performance: the ranks' kernels never wait on one another (the exchange
happens between steps).  Weak scaling makes every rank hold one periodic
copy of the grid, so the 2-rank metrics must equal the 1-rank ones."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest

from .conftest import REPO

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bench(workload, n, steps=3):
    env = dict(os.environ, WG_DIST_BACKEND="gloo", WG_FORCE_DEVICE="0", WG_FIXED_WARMUP="1")
    args = ["bench.py", "--gpus", str(n), "--steps", str(steps), "--warmup", "3", "--workload", workload,
            "--no-cpu-baseline"]
    if n > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr", "127.0.0.1", "--master-port", str(_port()), *args]
    else:
        cmd = [sys.executable, *args]
    out = subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("workload", ["lbm_c2", "swe_c3", "transport_c1"])
def test_two_ranks_weak_scaling(workload):
    one = _bench(workload, 1)
    two = _bench(workload, 2)
    assert two["n_gpus"] == 2 and two["scaling"] == "weak" and two["value"] > 0
    # two periodic copies: identical per-copy metrics
    assert two["compression_ratio"] == pytest.approx(one["compression_ratio"], rel=1e-12)
    assert two["compressed_bytes_per_step"] == pytest.approx(2 * one["compressed_bytes_per_step"], rel=1e-12)
    assert two["mass_drift"] <= 1e-12


@pytest.mark.parametrize("scheme", ["transport", "lbm"])
def test_peer_halos_across_processes(scheme):
    """Peer halo mode with real CUDA IPC between two processes (tests/peer_ipc_job.py)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "tests/peer_ipc_job.py", scheme, "4"]
    out = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    res = json.loads(lines[0])
    assert res["peer"] and res["equal"], res
