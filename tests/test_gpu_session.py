"""The fused compressed stencil loop (device session) against the C oracle's
run() — the reference's pipeline.hpp:129-305 restated — bit-exact in state,
compressed layout and integer metrics; mass within 1e-12 (summation order)."""
from __future__ import annotations

import ctypes as C
import json

import numpy as np
import pytest

from paper_2302_09883_b200 import abi, api

from .conftest import GOLDEN

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def compare_runs(a: api.RunResult, b: api.RunResult, mass_rtol=1e-12):
    assert len(a.rows) == len(b.rows)
    for ra, rb in zip(a.rows, b.rows):
        for k in ("step", "dense_bytes", "compressed_bytes", "nnz", "zeroed"):
            assert ra[k] == rb[k], (k, ra, rb)
        assert ra["time"] == rb["time"]
        assert ra["ratio"] == rb["ratio"]
        assert abs(ra["global_mass"] - rb["global_mass"]) <= mass_rtol * max(abs(rb["global_mass"]), 1.0)
    la, lb = a.grid.logical_view(), b.grid.logical_view()
    assert np.array_equal(bits(la), bits(lb)), f"{np.sum(la != lb)} logical cells differ"


def transport_cfg(nx, splits, levels, c, steps, mode="capped", **kw):
    cfg = api.RunConfig(scheme="transport", nx=nx, splits=splits, levels=levels,
                        spec=api.ThresholdSpec(mode, c), compute_l2=False, **kw)
    cfg.t_end = steps * cfg.cfl * (1.0 / (nx - 1)) / max(cfg.alpha, cfg.beta)
    return cfg


def test_c1_full_parity(product, oracle):
    """C1: 257^2 points, 8x8 patches of 33^2, L=4, capped 1e-3, 100 steps."""
    cfg = api.RunConfig(scheme="transport", nx=257, splits=(8, 8), levels=4, t_end=100 / 512,
                        spec=api.ThresholdSpec("capped", 1e-3), compute_l2=True)
    a = api.run(cfg, lib=product)
    b = api.run(cfg, lib=oracle)
    compare_runs(a, b)
    gold = json.loads((GOLDEN / "c1_transport.json").read_text())
    last = a.rows[-1]
    assert len(a.rows) == gold["steps"]
    assert last["nnz"] == gold["final"]["nnz"] and last["zeroed"] == gold["final"]["zeroed"]
    assert last["compressed_bytes"] == gold["final"]["compressed_bytes"]
    assert abs(a.summary["avg_ratio"] - gold["avg_ratio"]) <= 1e-12 * gold["avg_ratio"]
    assert abs(last["l2"] - gold["final"]["l2"]) <= 1e-12 * gold["final"]["l2"]


@pytest.mark.parametrize(
    "nx,splits,levels,c,mode,steps",
    [(33, (2, 2), 3, 0.01, "capped", 10),       # test_pipeline.cpp small_transport
     (65, (1, 1), 4, 1e-3, "capped", 5),        # single periodic patch
     (129, (2, 2), 4, 0.01, "capped", 20),      # acceptance transport_base (65^2 patches)
     (129, (2, 2), 2, 0.02, "accumulation", 8),
     (129, (8, 8), 3, 0.005, "constant", 8),    # 17^2 patches
     (257, (4, 4), 6, 1e-3, "capped", 6),       # L = k (non-conservative, still bit-exact)
     (65, (8, 8), 2, 0.05, "capped", 6),        # 9^2 patches
     (129, (2, 2), 0, 0.1, "capped", 4)],       # L = 0: nothing transforms, always raw
)
def test_transport_parity(product, oracle, nx, splits, levels, c, mode, steps):
    cfg = transport_cfg(nx, splits, levels, c, steps, mode)
    compare_runs(api.run(cfg, lib=product), api.run(cfg, lib=oracle))


def test_l2_every_step(product, oracle):
    """l2_error(assemble(grid), exact_transport(t)) of every row (pipeline.hpp:
    275-276) computed in the fused kernel; CUDA exp vs glibc exp and the
    summation order: relative 1e-12."""
    cfg = api.RunConfig(scheme="transport", nx=129, splits=(4, 4), levels=4, t_end=0.05,
                        spec=api.ThresholdSpec("capped", 1e-3), compute_l2=True)
    a, b = api.run(cfg, lib=product), api.run(cfg, lib=oracle)
    assert len(a.rows) == len(b.rows)
    for ra, rb in zip(a.rows, b.rows):
        assert abs(ra["l2"] - rb["l2"]) <= 1e-12 * rb["l2"], (ra["step"], ra["l2"], rb["l2"])


def test_zero_threshold_equals_no_compression(product):
    """test_pipeline.cpp:33-53 — c=0 keeps every patch raw (skip rule)."""
    a = api.run(transport_cfg(33, (2, 2), 3, 0.0, 12), lib=product)
    cfg = transport_cfg(33, (2, 2), 3, 0.0, 12)
    cfg.no_compression = True
    b = api.run(cfg, lib=product)
    assert all(r["zeroed"] == 0 for r in a.rows)
    assert all(r["compressed_bytes"] == 0 and r["ratio"] == 1.0 for r in b.rows)
    for ra, rb in zip(a.rows, b.rows):
        assert ra["global_mass"] == rb["global_mass"]
    assert np.array_equal(bits(a.grid.logical_view()), bits(b.grid.logical_view()))


def test_skip_rule_mixed_patches(product, oracle):
    """A threshold that zeroes nothing on some patches and something on
    others exercises the raw-patch kernel inside a compressed run."""
    cfg = transport_cfg(129, (4, 4), 3, 2e-5, 10)
    a, b = api.run(cfg, lib=product), api.run(cfg, lib=oracle)
    compare_runs(a, b)


def test_deterministic(product):
    cfg = transport_cfg(129, (4, 4), 4, 1e-3, 10)
    a, b = api.run(cfg, lib=product), api.run(cfg, lib=product)
    assert [r["global_mass"] for r in a.rows] == [r["global_mass"] for r in b.rows]
    assert np.array_equal(bits(a.grid.data), bits(b.grid.data))


def test_strict_mode_accepts_healthy_run(product):
    cfg = transport_cfg(33, (2, 2), 3, 0.01, 10, strict=True)
    api.run(cfg, lib=product)  # test_pipeline.cpp:73-77


def test_mass_conserved(product):
    cfg = transport_cfg(129, (2, 2), 4, 0.01, 40)
    r = api.run(cfg, lib=product)
    m0 = r.rows[0]["global_mass"]
    assert all(abs(x["global_mass"] - m0) <= 1e-10 * abs(m0) for x in r.rows)  # acceptance.cpp:197


def test_csr_bytes_accounting(product):
    """acceptance.cpp:251-255: bytes == 12 nnz + 4 * 66 * 4."""
    r = api.run(transport_cfg(129, (2, 2), 4, 0.01, 10), lib=product)
    assert all(x["compressed_bytes"] == 12 * x["nnz"] + 4 * 66 * 4 for x in r.rows)


def _session(product, cfg: api.RunConfig):
    c = cfg.to_c()
    s = abi.vp()
    product.check(product.wg_session_create(C.byref(c), None, None, C.byref(s)))
    return s


def test_session_csr_layout_bit_exact(product, oracle):
    """The stored CSR blocks equal csr_encode of the oracle's thresholded
    coefficients of the same state (index layout and values bit-exact)."""
    cfg = transport_cfg(129, (2, 2), 4, 1e-3, 3)
    s = _session(product, cfg)
    try:
        g0 = api.initial_state(cfg, lib=product)
        product.check(product.wg_session_upload(s, abi.dptr(g0.data)))
        dt = cfg.cfl / 128 / 0.9
        # oracle: one step by hand (sync, FV, DWT, threshold)
        ref = api.PatchGrid(g0.global_dims, g0.splits, 1, True, data=g0.data.copy())
        for _ in range(2):
            product.check(product.wg_session_step(s, dt))
            api.sync_ghosts(ref, lib=oracle)
            nxt = api.PatchGrid(ref.global_dims, ref.splits, 1, True, data=ref.data.copy())
            api.fv_step(ref, nxt, "transport", dt, 1 / 128, lib=oracle)
            ref = nxt
            for p in range(ref.npatch):
                blk = np.ascontiguousarray(ref.data[p, 0, 1:-1, 1:-1])
                cs = api.dwt_nd(blk, 4, lib=oracle)
                z = api.apply_threshold(cs, 4, cfg.spec, lib=oracle)
                assert z > 0
                ref.data[p, 0, 1:-1, 1:-1] = api.idwt_nd(cs + 0.0, 4, lib=oracle)
                want = api.csr_encode(cs, 65, 65, lib=oracle)
                nnz, raw = abi.u64(), abi.i32()
                product.check(product.wg_session_patch_csr(s, p, 0, None, None, None, C.byref(nnz), C.byref(raw)))
                assert raw.value == 0 and nnz.value == want.nnz()
                v = np.empty(nnz.value)
                col = np.empty(nnz.value, np.uint32)
                row = np.empty(66, np.uint32)
                product.check(product.wg_session_patch_csr(
                    s, p, 0, abi.dptr(v), col.ctypes.data_as(C.POINTER(abi.u32)),
                    row.ctypes.data_as(C.POINTER(abi.u32)), C.byref(nnz), C.byref(raw)))
                assert np.array_equal(bits(v), bits(want.v))
                assert np.array_equal(col, want.col) and np.array_equal(row, want.row)
    finally:
        product.wg_session_destroy(s)


def test_budget_overflow_fails_loudly(product):
    cfg = transport_cfg(129, (2, 2), 4, 1e-3, 2)
    cfg.store_budget_bytes = 64 * 1024  # smaller than the raw initial state
    s = _session(product, cfg)
    try:
        g0 = api.initial_state(cfg, lib=product)
        with pytest.raises(abi.OutOfMemoryError):
            product.check(product.wg_session_upload(s, abi.dptr(g0.data)))
    finally:
        product.wg_session_destroy(s)


# ---- D2Q9 LBM (builder-defined scheme on the reference's compression machinery) ----


def lbm_cfg(nx, splits, levels, c, steps, mode="capped", **kw):
    return api.RunConfig(scheme="lbm", nx=nx, splits=splits, levels=levels, lbm_steps=steps,
                         spec=api.ThresholdSpec(mode, c), **kw)


@pytest.mark.parametrize(
    "nx,splits,levels,c,steps",
    [(129, (4, 4), 4, 1e-3, 10),   # 33^2 patches
     (129, (2, 2), 4, 1e-3, 6),    # 65^2 patches (C2 patch shape)
     (129, (2, 2), 5, 1e-5, 5),    # L = 5 on 65^2, smallest threshold of the C2 sweep
     (65, (4, 4), 3, 1e-2, 8),     # 17^2 patches, largest threshold of the sweep
     (65, (1, 1), 3, 1e-4, 4),     # single periodic patch
     (129, (2, 2), 4, 0.0, 3)],    # nothing zeroed: every patch raw (skip rule)
)
def test_lbm_parity(product, oracle, nx, splits, levels, c, steps):
    cfg = lbm_cfg(nx, splits, levels, c, steps)
    compare_runs(api.run(cfg, lib=product), api.run(cfg, lib=oracle))


def test_lbm_no_compression_parity(product, oracle):
    cfg = lbm_cfg(129, (4, 4), 4, 1e-3, 6, no_compression=True)
    compare_runs(api.run(cfg, lib=product), api.run(cfg, lib=oracle))


def test_lbm_golden(product):
    gold = json.loads((GOLDEN / "small_lbm.json").read_text())
    r = api.run(lbm_cfg(129, (4, 4), 4, 1e-3, 20), lib=product)
    assert len(r.rows) == gold["steps"]
    for row, g in zip(r.rows, gold["rows"]):
        assert (row["nnz"], row["zeroed"], row["compressed_bytes"]) == (g["nnz"], g["zeroed"], g["compressed_bytes"])
    import hashlib
    assert hashlib.sha256(np.ascontiguousarray(r.grid.logical_view()).tobytes()).hexdigest() == gold["state_sha256"]


def test_lbm_mass_conserved(product):
    r = api.run(lbm_cfg(129, (2, 2), 4, 1e-3, 30), lib=product)
    m0 = r.rows[0]["global_mass"]
    assert all(abs(x["global_mass"] - m0) <= 1e-12 * abs(m0) for x in r.rows)


def test_lbm_device_initial_state(product, oracle):
    """wg_session_init_device: the shear-layer IC generated and compressed on
    the device (C4/C5 path) — close to the host IC (compression error and
    device libm), same mass, and it steps."""
    cfg = lbm_cfg(129, (4, 4), 4, 1e-4, 3)
    s = _session(product, cfg)
    try:
        product.check(product.wg_session_init_device(s))
        g = api.PatchGrid((129, 129), (4, 4), 9, True)
        product.check(product.wg_session_download(s, abi.dptr(g.data)))
        ic = api.initial_state(cfg, lib=oracle)
        diff = np.max(np.abs(g.logical_view() - ic.logical_view()))
        assert diff < 2e-3, diff
        m_dev = sum(api.global_mass(g, q, lib=oracle) for q in range(9))
        m_ic = sum(api.global_mass(ic, q, lib=oracle) for q in range(9))
        assert abs(m_dev - m_ic) <= 1e-12 * m_ic
        for _ in range(3):
            product.check(product.wg_session_step(s, 1.0))
        rows = (abi.MetricsRowC * 3)()
        n = abi.u64()
        product.check(product.wg_session_metrics(s, rows, 3, C.byref(n)))
        assert n.value == 3 and all(abs(r.global_mass - m_ic) <= 1e-11 * m_ic for r in rows)
    finally:
        product.wg_session_destroy(s)


def _run_session(product, cfg, host_grid, steps, dt=1.0):
    s = _session(product, cfg)
    try:
        product.check(product.wg_session_upload(s, abi.dptr(host_grid)))
        for _ in range(steps):
            product.check(product.wg_session_step(s, dt))
        info = abi.SessionInfoC()
        product.check(product.wg_session_info_get(s, C.byref(info)))
        out = np.zeros(info.npatch_local * info.components * (info.patch_n + 2) ** 2)
        product.check(product.wg_session_download(s, abi.dptr(out)))
        rows = (abi.MetricsRowC * steps)()
        n = abi.u64()
        product.check(product.wg_session_metrics(s, rows, steps, C.byref(n)))
        return out, [(r.nnz, r.zeroed, r.compressed_bytes) for r in rows]
    finally:
        product.wg_session_destroy(s)


def test_tiled_grid_copies_are_identical(product):
    """Weak-scaling geometry (wg_run_config::tile_rows): two periodic copies
    of the grid stacked along dim 0 evolve exactly like the single grid."""
    cfg = lbm_cfg(129, (4, 4), 4, 1e-3, 4)
    g0 = api.initial_state(cfg, lib=product)
    one, rows1 = _run_session(product, cfg, g0.data.reshape(-1).copy(), 4)
    cfg2 = lbm_cfg(129, (4, 4), 4, 1e-3, 4)
    cfg2.tile_rows = 2
    two, rows2 = _run_session(product, cfg2, np.concatenate([g0.data.reshape(-1)] * 2), 4)
    half = one.size
    assert np.array_equal(bits(two[:half]), bits(one)) and np.array_equal(bits(two[half:]), bits(one))
    assert all((a[0] * 2, a[1] * 2, a[2] * 2) == b for a, b in zip(rows1, rows2))


def test_pinned_upload_equals_pageable(product):
    import torch

    cfg = transport_cfg(129, (4, 4), 4, 1e-3, 3)
    g0 = api.initial_state(cfg, lib=product).data.reshape(-1).copy()
    pinned = torch.empty(g0.size, dtype=torch.float64, pin_memory=True)
    pinned.numpy()[:] = g0
    dt = cfg.cfl / 128 / 0.9
    a, ra = _run_session(product, cfg, g0, 3, dt)
    b, rb = _run_session(product, cfg, pinned.numpy(), 3, dt)
    assert np.array_equal(bits(a), bits(b)) and ra == rb


def test_lbm_directory_ends_on_page_boundary(product):
    """512^2 patches x 9 populations x 16 B = 36 MiB of directory, ending
    exactly on a 2 MiB page: a read past the last patch's entries faults
    (regression: idle threads of the last patch read entry 9)."""
    cfg = lbm_cfg(8193, (512, 512), 3, 1e-3, 2)
    s = _session(product, cfg)
    try:
        product.check(product.wg_session_init_device(s))
        for _ in range(2):
            product.check(product.wg_session_step(s, 1.0))
        product.check(product.wg_session_sync(s))
    finally:
        product.wg_session_destroy(s)


# ---- strict mode (pipeline.hpp:278-283) and RunSummary (pipeline.hpp:52-63) ----


@pytest.mark.parametrize("scheme", ["transport", "lbm"])
def test_strict_shared_cell_mismatch_raises(product, scheme):
    """assemble(grid, 0)'s check on the device: a shared boundary cell of
    component 0 that differs between its two owners beyond 1e-12 relative
    raises WG_CONSISTENCY; equal (or 1e-14-close) ones pass."""
    cfg = (transport_cfg(129, (2, 2), 4, 1e-3, 2) if scheme == "transport" else lbm_cfg(129, (2, 2), 4, 1e-3, 2))
    g0 = api.initial_state(cfg, lib=product)
    s = _session(product, cfg)
    try:
        product.check(product.wg_session_upload(s, abi.dptr(g0.data)))
        product.check(product.wg_session_check_shared(s, 1e-12))  # healthy
    finally:
        product.wg_session_destroy(s)
    bad = g0.data.copy()
    # patch 0's last logical column is patch 1's first (true index 65 vs 1)
    bad[0, 0, 10, 65] += 1e-6
    s = _session(product, cfg)
    try:
        product.check(product.wg_session_upload(s, abi.dptr(bad)))
        with pytest.raises(abi.ConsistencyError):
            product.check(product.wg_session_check_shared(s, 1e-12))
    finally:
        product.wg_session_destroy(s)
    close = g0.data.copy()
    close[0, 0, 10, 65] *= 1.0 + 1e-14
    s = _session(product, cfg)
    try:
        product.check(product.wg_session_upload(s, abi.dptr(close)))
        product.check(product.wg_session_check_shared(s, 1e-12))
    finally:
        product.wg_session_destroy(s)


@pytest.mark.parametrize("scheme", ["transport", "lbm", "swe"])
def test_strict_run_passes_and_summary_split(product, scheme):
    """strict run() (mass + shared cells every step) accepts a healthy run;
    the RunSummary phase split is populated and overhead() > 0."""
    if scheme == "transport":
        cfg = transport_cfg(129, (2, 2), 4, 1e-3, 6, strict=True)
    elif scheme == "lbm":
        cfg = lbm_cfg(129, (2, 2), 4, 1e-3, 6, strict=True)
    else:
        cfg = api.RunConfig(scheme="swe", nx=129, splits=(2, 2), levels=4, t_end=0.003,
                            spec=api.ThresholdSpec("constant", 5e-4), strict=True)
    r = api.run(cfg, lib=product)
    sm = r.summary
    assert sm["total_seconds"] > 0 and sm["step_seconds"] > 0
    assert sm["dwt_seconds"] > 0 and sm["threshold_seconds"] > 0 and sm["codec_seconds"] > 0
    parts = sm["step_seconds"] + sm["dwt_seconds"] + sm["threshold_seconds"] + sm["codec_seconds"]
    assert abs(parts - sm["total_seconds"]) <= 1e-9 + 1e-6 * sm["total_seconds"]
    overhead = (sm["total_seconds"] - sm["step_seconds"]) / sm["step_seconds"]  # RunSummary::overhead()
    assert overhead > 0
