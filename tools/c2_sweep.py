#!/usr/bin/env python
"""C2 as BASELINE.json states it: D2Q9 LBM, 1024^2, 64^2-cell patches, a
threshold sweep 1e-2..1e-5 with the error against the uncompressed run
(1000 steps per threshold plus an uncompressed run, relative
L2/Linf of rho and u, compression ratio, mass drift), on the device session.

usage: python tools/c2_sweep.py [--steps 1000] [--levels 4 5] [--out profiles/r1_c2_sweep.json]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

from paper_2302_09883_b200 import abi, api  # noqa: E402
from paper_2302_09883_b200.distributed import ShardInfo, ShardedSession  # noqa: E402

CX = np.array([0, 1, -1, 0, 0, 1, -1, 1, -1], dtype=np.float64)
CY = np.array([0, 0, 0, 1, -1, 1, -1, -1, 1], dtype=np.float64)


def run(lib, levels, c, steps, no_compression=False):
    cfg = api.RunConfig(scheme="lbm", nx=1025, splits=(16, 16), levels=levels, lbm_steps=steps,
                        spec=api.ThresholdSpec("capped", c), no_compression=no_compression, compute_l2=False)
    g = api.initial_state(cfg, lib=lib)
    s = ShardedSession(lib, cfg, ShardInfo(0, 1, 0, 16, 0), None)
    try:
        s.upload(g.data)
        s.sync()
        t0 = time.perf_counter()
        for _ in range(steps):
            s.step(1.0)
        s.sync()
        secs = time.perf_counter() - t0
        rows = s.rows()
        lib.check(lib.wg_session_download(s.handle, abi.dptr(g.data)))
    finally:
        s.close()
    f = g.logical_view()  # [patch][q][65][65]
    rho = f.sum(axis=1)
    ux = np.tensordot(CX, f, axes=([0], [1])) / rho
    uy = np.tensordot(CY, f, axes=([0], [1])) / rho
    m0, m1 = rows[0]["global_mass"], rows[-1]["global_mass"]
    return {"rho": rho, "ux": ux, "uy": uy, "glups": 1024 * 1024 * steps / secs / 1e9,
            "avg_ratio": float(np.mean([r["ratio"] for r in rows])), "mass_drift": abs(m1 - m0) / abs(m0)}


def rel(a, b):
    return {"l2": float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel())),
            "linf": float(np.max(np.abs(a - b)) / np.max(np.abs(b)))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--levels", type=int, nargs="+", default=[4, 5])
    ap.add_argument("--out", default=str(REPO / "profiles" / "r1_c2_sweep.json"))
    args = ap.parse_args()
    lib = abi.load_product()
    base = run(lib, 4, 0.0, args.steps, no_compression=True)
    out = {"config": "C2: D2Q9 1024^2, 16x16 patches of 65^2, capped thresholds, shear layer, "
                     f"{args.steps} steps; errors vs the uncompressed run of the same session code",
           "uncompressed": {"glups": base["glups"], "mass_drift": base["mass_drift"]}, "runs": []}
    for L in args.levels:
        for c in (1e-2, 1e-3, 1e-4, 1e-5):
            r = run(lib, L, c, args.steps)
            u = np.sqrt(r["ux"] ** 2 + r["uy"] ** 2)
            ub = np.sqrt(base["ux"] ** 2 + base["uy"] ** 2)
            e = {"levels": L, "c": c, "glups": r["glups"], "avg_ratio": r["avg_ratio"],
                 "mass_drift": r["mass_drift"], "rho": rel(r["rho"], base["rho"]), "u": rel(u, ub)}
            out["runs"].append(e)
            print(json.dumps(e), flush=True)
    Path(args.out).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
