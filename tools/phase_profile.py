#!/usr/bin/env python
"""Per-phase cycle breakdown of the fused step kernel (tuning builds with
-DWG_PHASE_TIMING: python -m paper_2302_09883_b200.build -DWG_PHASE_TIMING --variant=prof)."""
import argparse
import ctypes as C
import os
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
os.environ.setdefault("WG_PRODUCT_LIB", str(REPO / "paper_2302_09883_b200" / "libwavegrid_b200_prof.so"))

import bench  # noqa: E402
from paper_2302_09883_b200 import abi, api  # noqa: E402
from paper_2302_09883_b200.distributed import ShardInfo, ShardedSession  # noqa: E402

LBM_NAMES = {12: "end of patch (sums, reset)", 13: "D0 mbarrier wait", 14: "D0 masks + ghost gather",
             21: "D1 decode rows", 22: "D2 decode cols + stream", 23: "cluster sync (streamed)",
             24: "C collide", 25: "cluster sync (collided)", 26: "F1 col fwd + cluster sync", 27: "F2 row fwd + thr",
             28: "S scan + M1", 29: "alloc + M2", 30: "W CSR + cone rows", 31: "edge lines + patch sums"}
NAMES = {0: "decode rows+ghosts", 1: "decode cols", 2: "FV + mass", 3: "sync before fwd", 4: "fwd col DWT",
         5: "row DWT+thr+scan", 6: "alloc", 7: "CSR write + row inv", 8: "col recon+edges", 9: "raw store",
         10: "group sums", 11: "finalize"}
SWE_NAMES = {0: "decode rows+ghosts", 1: "decode cols", 2: "Godunov FV + mass", 4: "fwd col DWT",
             5: "row DWT+thr+scan", 6: "alloc", 7: "CSR write + row inv", 8: "col recon+edges",
             13: "store tile", 14: "wave speed", 9: "raw store", 11: "finalize"}
ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="transport_4k_p33")
ap.add_argument("--steps", type=int, default=10)
args = ap.parse_args()
w = bench.WORKLOADS[args.workload]
lib = abi.load_product()
lib.dll.wg_debug_phase_cycles.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.c_int32, C.c_int32]
cfg = bench.run_config(w, args.steps + 3)
dt = bench.transport_dt(cfg) if w["scheme"] == "transport" else 1.0
sess = ShardedSession(lib, cfg, ShardInfo(0, 1, 0, w["splits"][0], 0), None)
if w.get("streamed") or w.get("device_init"):  # budgeted grids: the device IC (same per-step work)
    sess.init_device()
else:
    sess.upload(api.initial_state(cfg, lib=lib).data)
for _ in range(3):
    sess.step(dt)
sess.sync()
buf = (C.c_uint64 * 32)()
lib.check(lib.dll.wg_debug_phase_cycles(sess.handle, buf, 32, 1))
for _ in range(args.steps):
    sess.step(dt)
sess.sync()
lib.check(lib.dll.wg_debug_phase_cycles(sess.handle, buf, 32, 0))
tot = sum(buf[:32])
ctas = sess.info  # noqa
print(f"{args.workload}: total thread0 cycles {tot:.3e} over {args.steps} steps")
for k in range(32):
    if buf[k]:
        nm = {"lbm": LBM_NAMES, "swe": SWE_NAMES}.get(w["scheme"], NAMES).get(k, "?")
        print(f"  {k:2d} {nm:26s} {100 * buf[k] / tot:5.1f}%")
sess.close()
