#!/usr/bin/env python
"""Benchmark of the compressed stencil loop (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload lbm_c4]
    python bench.py --impl reference ...      # the reference CPU path

A "step" is one pass of the hot path over the whole grid: ghost lines ->
decode -> scheme update -> DWT -> threshold -> CSR -> edge lines, for every
patch (pipeline.hpp:194-289).  The default workload is BASELINE.json
configs[3] (C4), the largest single-GPU configuration: D2Q9 LBM on 16384^2
cells in 64^2-cell patches (65^2 points), level 4, capped threshold 1e-3,
synthetic shear-layer initial state generated on the host (bit-identical to
the reference-style IC), under an 8 GiB store budget smaller than the 19.9 GB
raw state.  With N > 1 ranks (torchrun) the patch rows are sharded (strong
scaling) and the halo lines move over NCCL (or NVLink peer stores) every
step.

Prints ONE JSON line (rank 0).  Timing: CUDA events around every step on the
session stream, L2 flushed (a 256 MiB write) between timed steps outside the
events; max over ranks.  `roofline` uses the algorithmic bytes of SURVEY §8d
(2 m 8 B per cell-update, the uncompressed-equivalent state traffic).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

import numpy as np  # noqa: E402

from paper_2302_09883_b200 import abi, api  # noqa: E402

METRIC = "MLUPS (cell-updates/s) w/ compression @1/2/4/8 B200; HBM roofline %; compression ratio"

WORKLOADS = {
    # BASELINE.json configs[1] (C2)
    "lbm_c2": dict(scheme="lbm", components=9, nx=1025, splits=(16, 16), levels=4, c=1e-3, mode="capped",
                   scaling="weak"),
    # C2 with Codec::lz (codec.hpp:81-244): the device computes every block's LZ stream size
    # (the paper's higher ratios); the store itself stays CSR
    "lbm_c2_lz": dict(scheme="lbm", components=9, nx=1025, splits=(16, 16), levels=4, c=1e-3, mode="capped",
                      codec="lz", scaling="weak"),
    # C2 grid in 32^2-cell patches (occupancy study: 33-point lines need half the registers)
    "lbm_c2_p33": dict(scheme="lbm", components=9, nx=1025, splits=(32, 32), levels=4, c=1e-3, mode="capped",
                       scaling="weak"),
    # BASELINE.json configs[0] (C1): the reference's own CPU-runnable case
    "transport_c1": dict(scheme="transport", components=1, nx=257, splits=(8, 8), levels=4, c=1e-3, mode="capped"),
    # BASELINE.json configs[3] (C4): 16384^2 D2Q9 on one GPU; the raw f-field
    # (19.9 GB) exceeds the 8 GiB store budget: the host initial state (glibc,
    # bit-identical to the reference IC) streams through the device into step 1
    # (wg_session_step_host) and never enters the store.  N > 1: the shards'
    # initial state is generated and compressed on the device instead.
    "lbm_c4": dict(scheme="lbm", components=9, nx=16385, splits=(256, 256), levels=4, c=1e-3, mode="capped",
                   budget=8 << 30, streamed=True, scaling="strong"),
    # C4 / C2 at threshold 1e-5 (SURVEY §8d's sweep end): detail coefficients
    # survive (ratio ~52), the general decode path runs
    "lbm_c4_t1e5": dict(scheme="lbm", components=9, nx=16385, splits=(256, 256), levels=4, c=1e-5, mode="capped",
                        budget=8 << 30, streamed=True, scaling="strong"),
    "lbm_c2_t1e5": dict(scheme="lbm", components=9, nx=1025, splits=(16, 16), levels=4, c=1e-5, mode="capped",
                        scaling="weak"),
    # C4 with the device-generated initial state (the N > 1 path on one GPU)
    "lbm_c4_devinit": dict(scheme="lbm", components=9, nx=16385, splits=(256, 256), levels=4, c=1e-3,
                           mode="capped", budget=8 << 30, device_init=True, scaling="strong"),
    # BASELINE.json configs[4] (C5): 65536^2 D2Q9 (319 GB raw), sharded by patch
    # rows over the ranks; fits ONE B200 compressed
    "lbm_c5": dict(scheme="lbm", components=9, nx=65537, splits=(1024, 1024), levels=4, c=1e-3, mode="capped",
                   budget=24 << 30, device_init=True, scaling="strong"),
    # BASELINE.json configs[2] (C3): the reference's Riemann-type shock test —
    # SWE dam break, 4096^2 cells, 64^2-cell patches, constant c = 5e-4
    # (SURVEY §8d); t_end far beyond the timed steps, so every step is live
    "swe_c3": dict(scheme="swe", components=3, nx=4097, splits=(64, 64), levels=4, c=5e-4, mode="constant",
                   t_end=1.0, scaling="weak"),
    # C3-sized transport grid in 32^2-cell patches (C1 patch shape)
    "transport_4k_p33": dict(scheme="transport", components=1, nx=4097, splits=(128, 128), levels=4, c=1e-3, mode="capped"),
    # C3-sized transport grid (4096^2 cells, 64^2-cell patches)
    "transport_4k": dict(scheme="transport", components=1, nx=4097, splits=(64, 64), levels=4, c=1e-3, mode="capped"),
}

B_ALG = {"transport": 16, "swe": 48, "lbm": 144}  # bytes per cell-update, SURVEY §8d
# fp64 flops per cell-update, SURVEY §8d's count (transport ~49, D2Q9 ~430);
# SWE: the exact Riemann solves dominate (4 per cell, a few Newton iterations)
FLOPS_EST = {"transport": 49, "lbm": 430}


def data_label(w: dict) -> str:
    return {"lbm": "synthetic (shear-layer D2Q9 initial state)",
            "swe": "synthetic (reference dam-break initial state, pipeline.hpp:144-155)"}.get(
                w["scheme"], "synthetic (reference initial state, exact_transport at t=0)")


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_config(w: dict, steps: int) -> api.RunConfig:
    cfg = api.RunConfig(scheme=w["scheme"], nx=w["nx"], splits=tuple(w["splits"]), levels=w["levels"],
                        spec=api.ThresholdSpec(w["mode"], w["c"]), lbm_steps=steps,
                        compute_l2=w["scheme"] == "transport")  # run() computes l2 every step (pipeline.hpp:275-276)
    if w["scheme"] == "transport":
        cfg.t_end = steps * cfg.cfl * (1.0 / (w["nx"] - 1)) / max(cfg.alpha, cfg.beta)
    elif w["scheme"] == "swe":
        cfg.t_end = w.get("t_end", 1.0)
    cfg.store_budget_bytes = w.get("budget", 0)
    cfg.codec = w.get("codec", "csr")
    return cfg


def transport_dt(cfg: api.RunConfig) -> float:
    return cfg.cfl * (cfg.domain_length / (cfg.nx - 1)) / max(cfg.alpha, cfg.beta)


def peaks() -> dict:
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


# ---- clocks sampler (nvidia-smi during the timed region) -----------------------
_REASON_BITS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
    0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
    0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


class ClockSampler:
    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def count(self) -> int:
        return len(self.lines)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 3:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
                bits = int(parts[2], 16)
            except ValueError:
                continue
            for b, name in _REASON_BITS.items():
                if bits & b and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm),
                "sampled_during": "the timed steps" if not getattr(self, "extended", 0) else
                f"the timed steps and {self.extended} further untimed steps of the same workload"}


# ---- CPU baselines (oracles: the checker, timed only as the reported baseline) ---


def cpu_lib():
    ref = REPO / "oracle" / "_ref" / "libwg_ref.so"
    if ref.exists():
        return abi.Lib(ref), "reference"
    port = REPO / "oracle" / "libwg_oracle.so"
    if not port.exists():
        subprocess.run(["make", "-s", "-C", str(REPO / "oracle"), "c"], check=True)
    return abi.Lib(port), "port"


def cpu_run(w: dict, steps: int, threads: int):
    """Time the CPU implementation on `steps` steps of the workload; returns
    (MLUPS, seconds, kind, cores, rows, sample).  C4/C5 do not fit the CPU in
    minutes (268 M / 4.3 G cells per step): their per-cell work (65^2-point
    patches, L = 4, capped 1e-3) is timed on the C2 grid (1024^2) — declared
    in `sample` and by same_config = false."""
    name = w.get("_name", "")
    same = not (w.get("device_init") or w.get("streamed"))
    if not same:
        w = WORKLOADS["lbm_c2"]
    lib, kind = cpu_lib()
    cfg = run_config(w, steps)
    if w["scheme"] == "swe":
        # run() has no step cap: end the run after about `steps` CFL steps of
        # the initial state (dam break: vmax0 = sqrt(2 g); later dts shrink,
        # so the run takes at least that many steps — the rate counts them all)
        cfg.t_end = steps * cfg.cfl * (cfg.domain_length / (w["nx"] - 1)) / (2.0 * cfg.gravity) ** 0.5
    if w["scheme"] == "transport":
        cfg.compute_l2 = True  # run() computes the l2 diagnostic every step (pipeline.hpp:275-276)
    cfg.threads = threads if kind == "reference" else 1
    res = api.run(cfg, lib=lib)
    secs = res.summary["total_seconds"]
    cells = (w["nx"] - 1) ** 2
    if w["scheme"] == "lbm":
        # the reference has no LBM: the builder's D2Q9 on the
        # reference's own Patch / sync_ghosts / compression functions
        what = ("the builder's D2Q9 on the reference's Patch/sync_ghosts/compression functions "
                "(oracle/_ref/ref_shim.cpp, reference headers compiled unchanged)" if kind == "reference"
                else "the builder's D2Q9 in the C restatement (oracle/wg_oracle.c)")
        kind = "port"
    else:
        what = "run() of the reference headers (oracle/_ref)" if kind == "reference" else "run() of the C port"
    grid = f"{w['nx'] - 1}^2"
    sample = (f"{len(res.rows)} steps of the {grid} workload, {what}, {cfg.threads} threads, {secs:.1f} s"
              + ("" if same else f"; C2 grid standing in for {name} (same 65^2-point patches, L=4, capped 1e-3)"))
    return cells * len(res.rows) / secs / 1e6, secs, kind, cfg.threads, res.rows, sample, same


# ---- the reference arm -----------------------------------------------------------


def bench_reference(args, w: dict):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # the reference CPU path runs once, on rank 0
    threads = os.cpu_count() or 1
    if args.warmup:
        cpu_run(w, max(1, min(args.warmup, 2)), threads)
    mlups, secs, kind, cores, rows, sample, same = cpu_run(w, args.steps, threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": mlups, "unit": "MLUPS", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / len(rows),
        "higher_is_better": True, "scaling": w.get("scaling", "weak"), "vs_baseline": None, "dtype": "f64",
        "data": data_label(w), "config": config_json(args, w), "same_config": same,
        "compression_ratio": statistics.fmean(r["ratio"] for r in rows),
        "cpu_baseline": {"value": mlups, "unit": "MLUPS", "cores": cores, "kind": kind, "cpu": cpu_model(),
                         "sample": sample},
        "e2e": {"value": mlups, "unit": "MLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_json(args, w):
    n = (w["nx"] - 1) // w["splits"][0] + 1
    return {"workload": args.workload, "scheme": w["scheme"], "grid_cells": f"{w['nx'] - 1}x{w['nx'] - 1}",
            "patch_points": f"{n}x{n}", "patches": w["splits"][0] * w["splits"][1], "levels": w["levels"],
            "threshold": f"{w['mode']} c={w['c']}", "codec": w.get("codec", "csr"),
            "parallelism": f"patch-row shards x{args.gpus}"
                           + (" (weak: one periodic copy of the grid per rank)" if w.get("scaling", "weak") == "weak" else
                              " (strong: the grid split over the ranks)"),
            "halo_exchange": ("none (one shard)" if args.gpus == 1 else
                              "in-kernel NVLink peer stores (CUDA IPC; WG_PEER_HALOS=0: NCCL)"
                              if os.environ.get("WG_PEER_HALOS", "1") == "1" and w["scheme"] != "swe"
                              else "NCCL point-to-point between steps"),
            "l2": "flushed between timed steps (256 MiB write)"}


# ---- the B200 arm ----------------------------------------------------------------


def host_initial_state(lib, cfg, rb: int, re_: int, weak: bool, splits1: int, square_cfg):
    """This rank's initial grid buffer in page-locked memory, filled by the
    product's host IC (glibc libm: bit-identical to the reference IC,
    host threads over patch rows)."""
    import torch

    if weak:  # every rank's rows are one periodic copy of the square grid
        full = api.initial_state(square_cfg, lib=lib)
        pinned = torch.empty(full.data.size, dtype=torch.float64, pin_memory=True)
        pinned.numpy()[:] = full.data.reshape(-1)
        return pinned
    n = abi.u64()
    c = cfg.to_c()
    lib.check(lib.wg_run_grid_doubles(C.byref(c), C.byref(n)))
    per_row = n.value // cfg.splits[0]
    pinned = torch.empty(n.value, dtype=torch.float64, pin_memory=True)
    lib.check(lib.wg_run_initial_state(C.byref(c), abi.dptr(pinned.numpy())))
    if (rb, re_) != (0, cfg.splits[0]):
        own = torch.empty((re_ - rb) * per_row, dtype=torch.float64, pin_memory=True)
        own.copy_(pinned[rb * per_row: re_ * per_row])
        return own
    return pinned


def bench_b200(args, w: dict):
    import torch
    import torch.distributed as dist

    from paper_2302_09883_b200.distributed import ShardInfo, ShardedSession, collective_device, reduce_rows, shard_rows

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # WG_FORCE_DEVICE / WG_DIST_BACKEND=gloo: the N>1 orchestration run on one
    # GPU by tests/test_gpu_multiproc.py (correctness only; never a bench line)
    local = int(os.environ.get("WG_FORCE_DEVICE", local))
    torch.cuda.set_device(local)
    backend = os.environ.get("WG_DIST_BACKEND", "nccl")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
        # visible communicator: every rank's device, gathered over the process group
        names = [None] * world
        dist.all_gather_object(names, f"rank {rank}: cuda:{local} {torch.cuda.get_device_name(local)}")
        if rank == 0:
            nccl_v = ".".join(map(str, torch.cuda.nccl.version())) if backend == "nccl" else "-"
            print(f"[bench] process group {backend} (NCCL {nccl_v}) world {world}: " + "; ".join(names),
                  file=sys.stderr, flush=True)
    lib = abi.load_product()
    cfg = run_config(w, args.warmup + args.steps)
    dt = transport_dt(cfg) if w["scheme"] == "transport" else 1.0
    weak = w.get("scaling", "weak") == "weak"
    if weak:
        # weak scaling: the square problem replicated periodically along dim 0,
        # one copy per rank (identical work per rank; the halo exchange is real)
        cfg.tile_rows = world
    P0 = w["splits"][0] * (world if weak else 1)
    rb, re_ = shard_rows(P0, rank, world)
    shard = ShardInfo(rank, world, rb, re_, local)
    # a dedicated (non-default) stream: the session launches on it and the
    # CUDA events below are recorded on it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)

    # initial state: host (page-locked, bit-identical to the reference IC),
    # streamed into step 1 when the raw state exceeds the store budget (C4);
    # generated and compressed on the device for the sharded huge grids
    streamed = w.get("streamed", False) and world == 1
    device_init = w.get("device_init", False) or (w.get("streamed", False) and world > 1)
    host = None
    if not device_init:
        host = host_initial_state(lib, cfg, rb, re_, weak, w["splits"][1], run_config(w, 1)).numpy()

    sess = ShardedSession(lib, cfg, shard, stream.cuda_stream, dist if world > 1 else None)
    maybe_peer_halos(sess, cfg, dist, world)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    try:
        with ClockSampler(local) as clocks:
            if device_init:
                sess.init_device()
            elif not streamed:
                sess.upload(host)
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            # exactly W untimed warm-up steps (the first one streams the host
            # initial state in the C4 path)
            for k in range(args.warmup):
                if streamed and k == 0:
                    sess.step_host(host, dt)
                else:
                    sess.step(dt)
            sess.sync()
            warm_steps = args.warmup
            lib.check(lib.wg_session_profile(sess.handle, 1))
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            for e0, e1 in evs:
                flush.zero_()
                e0.record(stream)
                sess.step(dt)
                e1.record(stream)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            step_ms = [e0.elapsed_time(e1) for e0, e1 in evs]
            tot_ms = sum(step_ms)
            main_ms, launches = C.c_double(), abi.u64()
            lib.check(lib.wg_session_profile_read(sess.handle, C.byref(main_ms), C.byref(launches)))
            lib.check(lib.wg_session_profile(sess.handle, 0))
            rows = sess.rows()[: warm_steps + args.steps]
            # a timed region shorter than nvidia-smi's sampling period: the
            # same steps continue (untimed, not counted) until the clocks are
            # sampled under this load (clocks.sampled_during says so)
            clocks.extended = 0
            t_stop = time.perf_counter() + 1.0
            while world == 1 and clocks.count() < 3 and time.perf_counter() < t_stop:
                for _ in range(8):
                    sess.step(dt)
                sess.sync()
                clocks.extended += 8
        info = sess.info
        free_b, total_b = torch.cuda.mem_get_info(local)
        mem_used = total_b - free_b
        if world > 1:
            t = torch.tensor([tot_ms, main_ms.value], dtype=torch.float64,
                             device=collective_device(dist, f"cuda:{local}"))
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tot_ms, main_max = t.tolist()
            rows = reduce_rows(rows, dist, f"cuda:{local}")
        else:
            main_max = main_ms.value
        sess.close()

        # ---- end to end through the public API with host buffers -------------
        e2e = e2e_run(lib, cfg, shard, stream, host, args, dt, dist if world > 1 else None,
                      world if weak else 1, streamed)
    finally:
        sess.close()

    cells_global = (w["nx"] - 1) ** 2 * (world if weak else 1)
    value = cells_global * args.steps / (tot_ms * 1e-3) / 1e6
    pk = peaks()
    cells_local = info.cells_per_step
    launch_ms = main_ms.value / max(launches.value, 1)
    achieved = cells_local * B_ALG[w["scheme"]] / (launch_ms * 1e-3) / 1e9
    timed_rows = rows[warm_steps:]
    n = (w["nx"] - 1) // w["splits"][0] + 1
    kname = {"lbm": f"k_lbm_pair<{n},{w['levels']},STEP>", "swe": f"k_swe_step<{n},{w['levels']},STEP>"}.get(
        w["scheme"], f"k_patch_step<{n},{w['levels']},STEP>")
    line = {
        "metric": METRIC, "value": value, "unit": "MLUPS", "n_gpus": world, "steps": args.steps,
        "warmup": warm_steps, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
        "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": "f64",
        "data": data_label(w),
        "config": config_json(args, w),
        "compression_ratio": statistics.fmean(r["ratio"] for r in timed_rows),
        "compressed_bytes_per_step": statistics.fmean(r["compressed_bytes"] for r in timed_rows),
        "mass_drift": abs(timed_rows[-1]["global_mass"] - rows[0]["global_mass"]) / abs(rows[0]["global_mass"]),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / pk["hbm_gbs"], "traffic": traffic_from_profiles(args.workload),
                     "kernel": kname,
                     "algorithmic_bytes_per_launch": cells_local * B_ALG[w["scheme"]],
                     "avg_launch_ms": launch_ms, "peak_source": pk["source"],
                     "step_share": main_max / tot_ms if tot_ms else None},
        "e2e": e2e,
        "compute_ceiling": compute_ceiling(lib, w, value / world),  # per GPU
        # one fused kernel launch per step; Codec::lz adds the LZ-size pass
        # (k_lz_sizes, which also writes the step's row); the peer halo mode
        # adds its device-side wait and signal; transport adds the l2 pass
        "gpu_launches": args.steps * ((2 if w.get("codec") == "lz" else 1) + (2 if sess.peer else 0)
                                      + (1 if cfg.compute_l2 and w["scheme"] == "transport" else 0)),
        "clocks": clocks.summary(),
        "device_bytes": info.device_bytes,
        "device_mem_used_bytes": mem_used,
        "raw_state_bytes": 8 * w["components"] * (w["nx"] - 1) ** 2 if "components" in w else None,
        "initial_state": ("device-generated (CUDA libm, not bit-pinned)" if device_init else
                          "host glibc IC (bit-identical to the reference), streamed into step 1"
                          if streamed else "host glibc IC (bit-identical to the reference), uploaded"),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # bounded sample: calibrate on a few steps, then about 12 s of CPU work
        s0 = cpu_run(w, 3, os.cpu_count() or 1)[1]
        cpu_steps = args.cpu_steps or int(max(3, min(2000, 12.0 / max(s0 / 3, 1e-6))))
        mlups, secs, kind, cores, crow, sample, same = cpu_run(w, cpu_steps, os.cpu_count() or 1)
        line["cpu_baseline"] = {"value": mlups, "unit": "MLUPS", "cores": cores, "kind": kind, "cpu": cpu_model(),
                                "sample": sample, "same_config": same}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def compute_ceiling(lib, w, value_mlups):
    """The fp64 ceiling next to the HBM roofline: measured DFMA
    throughput of this GPU and, with SURVEY's flop count per cell-update,
    the compute-bound cell rate and this run's fraction of it."""
    t = C.c_double()
    lib.check(lib.wg_dev_fp64_probe(1 << 16, C.byref(t)))
    out = {"fp64_tflops_measured": t.value, "probe": "8 independent DFMA chains/thread, 8 CTAs x 256 per SM"}
    fl = FLOPS_EST.get(w["scheme"])
    if fl:
        ceil = t.value * 1e12 / fl / 1e6
        out.update({"flops_per_cell_estimate": fl, "ceiling_mlups": ceil, "frac": value_mlups / ceil})
    return out


def e2e_run(lib, cfg, shard, stream, host, args, dt, dist, copies=1, streamed=False):
    """Same metric through the public API with host buffers: inside the timed
    region the host initial state goes in from page-locked memory (streamed
    into step 1 in the C4 path), every step's metrics row comes back, and the
    final decoded state is read back into the host grid buffer."""
    import torch

    from paper_2302_09883_b200.distributed import ShardedSession, collective_device

    sess = ShardedSession(lib, cfg, shard, stream.cuda_stream, dist)
    maybe_peer_halos(sess, cfg, dist, shard.world)
    row_buf = torch.empty(args.steps * C.sizeof(abi.MetricsRowC), dtype=torch.uint8, pin_memory=True)
    out = None if host is None else host  # the state read back overwrites the (consumed) input buffer
    try:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if host is None:
            sess.init_device()
        elif not streamed:
            sess.upload(host)
        rowsz = C.sizeof(abi.MetricsRowC)
        for k in range(args.steps):
            if streamed and k == 0:
                sess.step_host(host, dt)
            else:
                sess.step(dt)
            # + the step's metrics row read back (async D2H into page-locked memory)
            lib.check(lib.wg_session_last_row_async(sess.handle, C.c_void_p(row_buf.data_ptr() + k * rowsz)))
        if out is not None:
            sess.download(out)
        torch.cuda.synchronize()
        secs = time.perf_counter() - t0
        if dist:
            t = torch.tensor([secs], dtype=torch.float64, device=collective_device(dist, f"cuda:{shard.device}"))
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            secs = t.item()
        got = (abi.MetricsRowC * args.steps).from_buffer_copy(row_buf.numpy().tobytes())
        assert all(r.step > 0 for r in got), "e2e: metrics rows not read back"
    finally:
        sess.close()
    cells = (cfg.nx - 1) ** 2 * copies
    row_b = C.sizeof(abi.MetricsRowC)
    if host is None:
        return {"value": cells * args.steps / secs / 1e6, "unit": "MLUPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": row_b, "seconds": secs,
                "note": "initial state generated and compressed on the device inside the timed region; "
                        "every step's metrics row read back (async D2H into page-locked memory)"}
    return {"value": cells * args.steps / secs / 1e6, "unit": "MLUPS",
            "h2d_bytes_per_step": host.nbytes / args.steps,
            "d2h_bytes_per_step": (host.nbytes + args.steps * row_b) / args.steps, "seconds": secs,
            "note": ("host initial state (page-locked) " + ("streamed into step 1" if streamed else "uploaded")
                     + f" and the final decoded state read back, {args.steps} steps, inside the timed region "
                       "(bytes amortised per step); every step's metrics row read back asynchronously")}


def peer_halos_wanted(cfg, dist, world: int) -> bool:
    """Peer halo mode (default at N > 1 over NCCL; WG_PEER_HALOS=0 selects the
    NCCL point-to-point exchange between steps): the step kernels store the
    halo lines into the neighbours' halo slots over NVLink (CUDA IPC)."""
    return (world > 1 and os.environ.get("WG_PEER_HALOS", "1") == "1" and cfg.scheme != "swe"
            and dist is not None and dist.get_backend() == "nccl")


def maybe_peer_halos(sess, cfg, dist, world: int) -> None:
    if peer_halos_wanted(cfg, dist, world):
        sess.connect_peers()


def traffic_from_profiles(workload: str):
    p = REPO / "profiles" / "traffic.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get(workload)
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=None,
                    help="default: lbm_c4 (BASELINE configs[3]) at N=1, lbm_c5 (configs[4], the grid split "
                         "over the ranks, peer halos) at N>1")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=0, help="CPU baseline steps (0: ~12 s of work)")
    args = ap.parse_args()
    if args.impl == "b200":
        args.warmup = max(args.warmup, 3)  # timing rule: at least 3 untimed warm-up steps
    if args.workload is None:
        args.workload = "lbm_c4" if args.gpus == 1 else "lbm_c5"
    w = dict(WORKLOADS[args.workload])
    w["_name"] = args.workload
    if args.impl == "reference":
        bench_reference(args, w)
    else:
        bench_b200(args, w)


if __name__ == "__main__":
    main()
