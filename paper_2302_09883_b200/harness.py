"""The reference's file and experiment harness around the hot path
(SURVEY §8f-2/3): WGRD snapshots (patchgrid.hpp:317-376), the WGC1
container writer (codec.hpp:364-391), transform_file / restore_file
(pipeline.hpp:311-337), sweep (pipeline.hpp:339-401) and the discontinuous
demo (pipeline.hpp:405-460).

Host-side orchestration only: every transform, threshold and codec call goes
through the C ABI of `lib` (the sm_100a product by default, so the compute
runs on the GPU's per-op kernels; the oracles in the tests).  Files are
written with Codec::csr; sweep and run accept Codec::lz (device-computed LZ
sizes, metrics only).
"""
from __future__ import annotations

import math
import os
import struct
from dataclasses import dataclass, field, replace
from pathlib import Path

import numpy as np

from . import abi, api

# ---- WGRD (patchgrid.hpp:317-376) ---------------------------------------------


def save_wgrd(path, comps) -> None:
    """save_wgrd: "WGRD", u32 version 1, u32 ndims, u32 dims[], u32 ncomp,
    then every component's values (f64, row-major)."""
    comps = [np.ascontiguousarray(c, dtype=np.float64) for c in comps]
    if not comps:
        raise ValueError("save_wgrd: no components")
    dims = comps[0].shape
    if any(c.shape != dims for c in comps):
        raise ValueError("save_wgrd: component dims differ")
    with open(path, "wb") as f:
        f.write(b"WGRD" + struct.pack("<II", 1, len(dims)) + struct.pack("<" + "I" * len(dims), *dims))
        f.write(struct.pack("<I", len(comps)))
        for c in comps:
            f.write(c.astype("<f8").tobytes())


def load_wgrd(path) -> list:
    with open(path, "rb") as f:
        if f.read(4) != b"WGRD":
            raise abi.CorruptStreamError("not a WGRD file")

        def u32():
            b = f.read(4)
            if len(b) != 4:
                raise abi.CorruptStreamError("truncated WGRD file")
            return struct.unpack("<I", b)[0]

        if u32() != 1:
            raise abi.CorruptStreamError("unsupported WGRD version")
        nd = u32()
        dims = tuple(u32() for _ in range(nd))
        nc = u32()
        n = int(np.prod(dims))
        out = []
        for _ in range(nc):
            b = f.read(8 * n)
            if len(b) != 8 * n:
                raise abi.CorruptStreamError("truncated WGRD file")
            out.append(np.frombuffer(b, dtype="<f8").reshape(dims).copy())
    return out


def assemble(grid: api.PatchGrid, comp: int) -> np.ndarray:
    """assemble(grid, comp) (patchgrid.hpp:203-242): the global logical field
    (shared patch-boundary points taken from the later patch; they agree)."""
    gd = grid.global_dims
    out = np.empty(gd)
    n = grid.logical
    lv = grid.logical_view()
    for p in range(grid.data.shape[0]):
        idx = np.unravel_index(p, grid.splits)
        sl = tuple(slice(k * (ni - 1), k * (ni - 1) + ni) for k, ni in zip(idx, n))
        out[sl] = lv[p, comp]
    return out


# ---- WGC1 writer (codec.hpp:364-391) --------------------------------------------


def encode_patch(arrays, dims, levels: int, codec: int = 1, lib=None) -> api.CompressedPatch:
    """encode_patch (codec.hpp:285-306) for Codec::csr: rows = prod of the
    leading dims, cols = the last."""
    if codec != 1:
        raise ValueError("Codec::lz is out of scope (SURVEY §8f-1)")
    rows = int(np.prod(dims[:-1])) if len(dims) > 1 else 1
    cols = int(dims[-1])
    blocks = [api.csr_encode(np.asarray(a).reshape(-1), rows, cols, lib=lib) for a in arrays]
    return api.CompressedPatch(1, tuple(dims), len(arrays), int(levels), blocks, [])


def save_wgc(f, p: api.CompressedPatch) -> None:
    f.write(b"WGC1" + struct.pack("<II", p.codec, len(p.dims)) + struct.pack("<" + "I" * len(p.dims), *p.dims))
    f.write(struct.pack("<II", p.components, p.levels))
    if p.codec != 1:
        raise ValueError("Codec::lz is out of scope (SURVEY §8f-1)")
    for b in p.csr:
        f.write(struct.pack("<II", b.rows, b.cols))
        for arr, dt in ((b.v, "<f8"), (b.col, "<u4"), (b.row, "<u4")):
            a = np.ascontiguousarray(arr, dtype=dt)
            f.write(struct.pack("<Q", a.size))
            f.write(a.tobytes())


# ---- transform_file / restore_file (pipeline.hpp:311-337) -----------------------


def transform_file(inp, levels: int, spec: api.ThresholdSpec, codec: int, chunk_size: int, out, lib=None) -> None:
    comps = load_wgrd(inp)
    dims = comps[0].shape
    arrays = []
    for c in comps:
        cs = api.dwt_nd(c, levels, lib=lib)  # WaveletPlan::validate inside
        api.apply_threshold(cs, levels, spec, lib=lib)
        arrays.append(cs)
    with open(out, "wb") as f:
        save_wgc(f, encode_patch(arrays, dims, levels, codec, lib=lib))


def restore_file(inp, out, lib=None) -> None:
    with open(inp, "rb") as f:
        p = api.load_wgc(f)
    arrays = api.decode_patch(p, lib=lib)
    comps = [api.idwt_nd(a.reshape(p.dims), p.levels, lib=lib) for a in arrays]
    save_wgrd(out, comps)


# ---- sweep (pipeline.hpp:339-401) ------------------------------------------------


@dataclass
class SweepConfig:
    base: api.RunConfig
    thresholds: list = field(default_factory=list)
    levels: list = field(default_factory=list)
    codecs: list = field(default_factory=lambda: [1])
    out_dir: str = ""


@dataclass
class SweepEntry:
    threshold: float
    level: int
    codec: int
    avg_ratio: float
    final_l2: float
    metrics_file: str


def sweep(cfg: SweepConfig, lib=None) -> list:
    if cfg.out_dir:
        os.makedirs(cfg.out_dir, exist_ok=True)
    table = []
    for codec in cfg.codecs:
        cname = {1: "csr", 2: "lz"}[codec]
        for level in cfg.levels:
            for c in cfg.thresholds:
                name = "run_%s_L%d_c%s.csv" % (cname, level, _fmt_g(c))
                rc = replace(cfg.base, levels=level, spec=replace(cfg.base.spec, c=c), codec=cname,
                             metrics_path=str(Path(cfg.out_dir) / name) if cfg.out_dir else name)
                r = api.run(rc, lib=lib)
                table.append(SweepEntry(c, level, codec, r.summary["avg_ratio"],
                                        r.rows[-1]["l2"] if r.rows else 0.0, rc.metrics_path))
    if cfg.out_dir:
        with open(Path(cfg.out_dir) / "summary.csv", "w") as f:
            f.write("codec,level,threshold,avg_ratio,final_l2_error,metrics_file\n")
            for e in table:
                f.write("%s,%d,%.17g,%.17g,%.17g,%s\n" % ({1: "csr", 2: "lz"}[e.codec], e.level, e.threshold,
                                                          e.avg_ratio, e.final_l2, e.metrics_file))
    return table


def _fmt_g(x: float) -> str:
    """printf("%g") (the sweep file names)."""
    return "%g" % x


# ---- demo_discontinuous (pipeline.hpp:405-460) -----------------------------------


@dataclass
class DemoReport:
    total: int
    nonzeros: int
    coefficient_ratio: float
    mass_before: float
    mass_after: float


def _trapezoid_mass_nd(f: np.ndarray) -> float:
    """trapezoid_mass_nd (wavelet.hpp:253-270): reduce the last dimension
    first with end weights 1/2."""
    x = np.asarray(f, dtype=np.float64)
    while x.ndim:
        w = np.ones(x.shape[-1])
        w[0] = w[-1] = 0.5
        s = np.zeros(x.shape[:-1])
        for k in range(x.shape[-1]):  # sequential, like the reference's loop
            s = s + w[k] * x[..., k]
        x = s
    return float(x)


def demo_discontinuous(out_dir: str = "", threshold: float = 0.2, lib=None) -> DemoReport:
    n = 129
    f = np.empty((n, n))
    for i in range(n):  # the C library's exp/sin (math.*), as the reference samples it
        for j in range(n):
            x, y = i / n, j / n
            stp = 1.0 if (y - x * x) >= 0.0 else 2.0
            f[i, j] = math.exp(x - y) * math.sin(2.0 * math.pi * (x + y)) * stp
    cs = api.dwt_nd(f, 6, lib=lib)
    api.apply_threshold(cs, 6, api.ThresholdSpec("constant", threshold), lib=lib)
    nz = int(np.count_nonzero(cs))
    rec = api.idwt_nd(cs, 6, lib=lib)
    rep = DemoReport(f.size, nz, f.size / nz if nz else 0.0, _trapezoid_mass_nd(f), _trapezoid_mass_nd(rec))
    if out_dir:
        os.makedirs(out_dir, exist_ok=True)
        save_wgrd(Path(out_dir) / "original.wgrd", [f])
        save_wgrd(Path(out_dir) / "reconstructed.wgrd", [rec])
        with open(Path(out_dir) / "report.txt", "w") as fh:
            fh.write(f"total coefficients: {rep.total}\nnonzero coefficients: {rep.nonzeros}\n"
                     f"coefficient-count ratio: {rep.coefficient_ratio:g}\nmass before: {rep.mass_before:g}\n"
                     f"mass after: {rep.mass_after:g}\n")
    return rep


# ---- run() with snapshots / observer (pipeline.hpp:160-181, 285-288) -------------


def run_observed(cfg: api.RunConfig, snapshot_times=(), snapshot_prefix: str = "", observer=None, lib=None):
    """run(RunConfig) driven step by step through the device session, for the
    harness features that need the state between steps: WGRD snapshots at
    `snapshot_times` (file `<prefix>t%.3f.wgrd`, the t = 0 one included) and
    `observer(grid, row)` after every step.  Each snapshot/observation
    decodes the compressed store to the host; the steps themselves are the
    same fused launches as run()."""
    import ctypes as C

    from .distributed import ShardInfo, ShardedSession

    L = api._lib(lib)
    if not hasattr(L, "wg_session_create"):
        raise ValueError("run_observed needs the device library (wg_session_*)")
    grid = api.initial_state(cfg, lib=L)
    P0 = cfg.splits[0]
    sess = ShardedSession(L, cfg, ShardInfo(0, 1, 0, P0, 0), None)
    done = [False] * len(snapshot_times)
    m = grid.components

    def snapshot(t):
        need = [s for s, ts in enumerate(snapshot_times) if not done[s] and t >= ts - 1e-9]
        if not need:
            return
        L.check(L.wg_session_download(sess.handle, api.abi.dptr(grid.data)))
        comps = [assemble(grid, c) for c in range(m)]
        for s in need:
            done[s] = True
            save_wgrd(f"{snapshot_prefix}t{snapshot_times[s]:.3f}.wgrd", comps)

    try:
        sess.upload(grid.data)
        snapshot(0.0)
        if cfg.scheme == "transport":
            dx = cfg.domain_length / (cfg.nx - 1)
            dt0 = cfg.cfl * dx / max(cfg.alpha, cfg.beta)  # cfl_dt, solver.hpp:235-241
            dts, t = [], 0.0
            while t < cfg.t_end - 1e-15:
                dt = min(dt0, cfg.t_end - t)
                dts.append(dt)
                t += dt
        elif cfg.scheme == "lbm":
            dts = [1.0] * cfg.lbm_steps
        else:
            dts = None  # SWE: the device clock decides; step until it stops
        k = 0
        while True:
            if dts is not None and k == len(dts):
                break
            sess.step(dts[k] if dts is not None else 1.0)
            n = api.abi.u64()
            L.check(L.wg_session_metrics(sess.handle, None, 0, C.byref(n)))
            if n.value == k:  # SWE: t_end reached, the launch was a no-op
                break
            k += 1
            row = sess.last_row()
            snapshot(row["time"])
            if observer is not None:
                L.check(L.wg_session_download(sess.handle, api.abi.dptr(grid.data)))
                observer(grid, row)
        rows = sess.rows()
        L.check(L.wg_session_download(sess.handle, api.abi.dptr(grid.data)))
    finally:
        sess.close()
    ratios = [r["ratio"] for r in rows]
    summary = {"avg_ratio": sum(ratios) / len(ratios) if ratios else 1.0, "steps": len(rows),
               "t_final": rows[-1]["time"] if rows else 0.0}
    return api.RunResult(rows, summary, grid, summary["t_final"])
