#!/usr/bin/env python
"""Minimal step driver for ncu captures (no timing, no CPU baseline):

    python tools/prof_step.py [--workload lbm_c2] [--steps 6]

Creates a device session for a bench.py workload, uploads (or device-
generates) the initial state and runs the steps on the session stream.
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2302_09883_b200 import abi, api  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="lbm_c2")
    ap.add_argument("--steps", type=int, default=6)
    args = ap.parse_args()
    w = bench.WORKLOADS[args.workload]
    lib = abi.load_product()
    cfg = bench.run_config(w, args.steps)
    dt = bench.transport_dt(cfg) if w["scheme"] == "transport" else 1.0
    c = cfg.to_c()
    s = abi.vp()
    lib.check(lib.wg_session_create(C.byref(c), None, None, C.byref(s)))
    try:
        if w.get("device_init"):
            lib.check(lib.wg_session_init_device(s))
        else:
            g0 = api.initial_state(bench.run_config(w, 1), lib=lib)
            lib.check(lib.wg_session_upload(s, abi.dptr(np.ascontiguousarray(g0.data))))
        for _ in range(args.steps):
            lib.check(lib.wg_session_step(s, dt))
        lib.check(lib.wg_session_sync(s))
        row = abi.MetricsRowC()
        lib.check(lib.wg_session_last_row(s, C.byref(row)))
        print(f"ok: step {row.step} ratio {row.ratio:.3f} nnz {row.nnz} mass {row.global_mass!r}")
    finally:
        lib.wg_session_destroy(s)


if __name__ == "__main__":
    main()
