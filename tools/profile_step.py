#!/usr/bin/env python
"""Run a few steps of a bench workload through the device session (no timing
logic, no CPU baseline): the command profiled by ncu for profiles/."""
import argparse
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

import bench  # noqa: E402
from paper_2302_09883_b200 import abi, api  # noqa: E402
from paper_2302_09883_b200.distributed import ShardInfo, ShardedSession  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="lbm_c2", choices=sorted(bench.WORKLOADS))
ap.add_argument("--steps", type=int, default=4)
args = ap.parse_args()
w = bench.WORKLOADS[args.workload]
lib = abi.load_product()
cfg = bench.run_config(w, args.steps)
dt = bench.transport_dt(cfg) if w["scheme"] == "transport" else 1.0
grid = api.initial_state(cfg, lib=lib)
sess = ShardedSession(lib, cfg, ShardInfo(0, 1, 0, w["splits"][0], 0), None)
sess.upload(grid.data)
for _ in range(args.steps):
    sess.step(dt)
sess.sync()
r = sess.rows()[-1]
print(f"{args.workload}: {args.steps} steps, ratio {r['ratio']:.2f}, nnz {r['nnz']}, mass {r['global_mass']:.15g}")
sess.close()
