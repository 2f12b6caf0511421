"""The fused shallow-water step (k_swe_step, swe_kernels.cuh) with its
device-side clock, against the C oracle's run() for Scheme::swe
(pipeline.hpp:129-305, solver.hpp:74-258).

Parity statement: the device squares the Newton start of solve_hstar by a
multiplication where the reference calls glibc pow(x, 2) (solver.hpp:112);
the two can differ by an ulp.  The product is therefore checked BIT-EXACT
against oracle/libwg_oracle_sq.so (the same restatement with b * b), and
against the reference-arithmetic oracle (pow) and the reference golden either
bit-exact or — should an ulp ever propagate — within SWE_TOL of the state.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json

import numpy as np
import pytest

from paper_2302_09883_b200 import abi, api

from .conftest import GOLDEN
from .test_gpu_session import bits, compare_runs

pytestmark = pytest.mark.gpu

SWE_TOL = 1e-9  # max |state difference| vs the pow() oracle (depths ~1-2)


def swe_cfg(nx, splits, levels, c, t_end, mode="constant", **kw):
    return api.RunConfig(scheme="swe", nx=nx, splits=splits, levels=levels, t_end=t_end,
                         spec=api.ThresholdSpec(mode, c), **kw)


def close_runs(a: api.RunResult, b: api.RunResult):
    assert len(a.rows) == len(b.rows)
    for ra, rb in zip(a.rows, b.rows):
        assert abs(ra["time"] - rb["time"]) <= 1e-12 * rb["time"]
    assert np.max(np.abs(a.grid.logical_view() - b.grid.logical_view())) <= SWE_TOL


def test_swe_golden(product):
    """test_pipeline.cpp small SWE case: 33^2, 2x2 patches, L=3, constant 5e-4."""
    gold = json.loads((GOLDEN / "small_swe.json").read_text())
    r = api.run(swe_cfg(33, (2, 2), 3, 5e-4, 0.05), lib=product)
    assert len(r.rows) == gold["steps"]
    last = r.rows[-1]
    assert (last["nnz"], last["zeroed"], last["compressed_bytes"]) == (
        gold["final"]["nnz"], gold["final"]["zeroed"], gold["final"]["compressed_bytes"])
    assert abs(r.summary["avg_ratio"] - gold["avg_ratio"]) <= 1e-12 * gold["avg_ratio"]
    assert hashlib.sha256(np.ascontiguousarray(r.grid.logical_view()).tobytes()).hexdigest() == gold["state_sha256"]


@pytest.mark.parametrize(
    "nx,splits,levels,c,mode,t_end",
    [(33, (2, 2), 3, 5e-4, "constant", 0.05),   # 17^2 patches (golden case)
     (129, (4, 4), 4, 5e-4, "constant", 0.02),  # 33^2 patches
     (129, (2, 2), 4, 1e-3, "capped", 0.01),    # 65^2 patches (C3 patch shape)
     (129, (2, 2), 6, 5e-4, "constant", 0.005), # L = k on 65^2
     (65, (8, 8), 2, 1e-3, "accumulation", 0.02),  # 9^2 patches
     (65, (1, 1), 4, 1e-3, "constant", 0.02),   # single periodic patch
     (65, (2, 2), 0, 1e-3, "constant", 0.01),   # L = 0: always raw
     (129, (2, 2), 4, 0.0, "constant", 0.01)],  # c = 0: nothing zeroed, skip rule
)
def test_swe_parity(product, oracle_sq, oracle, nx, splits, levels, c, mode, t_end):
    cfg = swe_cfg(nx, splits, levels, c, t_end, mode)
    a = api.run(cfg, lib=product)
    compare_runs(a, api.run(cfg, lib=oracle_sq))
    close_runs(a, api.run(cfg, lib=oracle))


def test_swe_no_compression_parity(product, oracle_sq):
    cfg = swe_cfg(129, (4, 4), 4, 5e-4, 0.01, no_compression=True)
    compare_runs(api.run(cfg, lib=product), api.run(cfg, lib=oracle_sq))


def test_swe_mass_conserved(product):
    """C3's metric: relative global mass drift of h over the run (the 5/3
    lifting with L < k conserves it to round-off)."""
    r = api.run(swe_cfg(257, (4, 4), 4, 5e-4, 0.02), lib=product)
    m0 = r.rows[0]["global_mass"]
    assert max(abs(x["global_mass"] - m0) for x in r.rows) <= 1e-12 * m0


def test_swe_strict_mode(product):
    cfg = swe_cfg(129, (2, 2), 4, 1e-3, 0.005, strict=True)
    api.run(cfg, lib=product)


def _session(product, cfg):
    c = cfg.to_c()
    s = abi.vp()
    product.check(product.wg_session_create(C.byref(c), None, None, C.byref(s)))
    return s


def test_swe_session_clock(product, oracle_sq):
    """wg_session_step ignores dt for SWE: each call runs one step with the
    device's CFL dt, and calls past t_end are no-ops."""
    cfg = swe_cfg(65, (2, 2), 3, 5e-4, 0.01)
    ref = api.run(cfg, lib=oracle_sq)
    g0 = api.initial_state(cfg, lib=oracle_sq)
    s = _session(product, cfg)
    try:
        product.check(product.wg_session_upload(s, abi.dptr(g0.data)))
        for _ in range(len(ref.rows) + 5):
            product.check(product.wg_session_step(s, 123.0))
        n = abi.u64()
        rows = (abi.MetricsRowC * (len(ref.rows) + 5))()
        product.check(product.wg_session_metrics(s, rows, len(ref.rows) + 5, C.byref(n)))
        assert n.value == len(ref.rows)
        for r, g in zip(rows[: n.value], ref.rows):
            assert (r.step, r.time, r.nnz, r.zeroed) == (g["step"], g["time"], g["nnz"], g["zeroed"])
        out = api.PatchGrid((65, 65), (2, 2), 3, True)
        product.check(product.wg_session_download(s, abi.dptr(out.data)))
        assert np.array_equal(bits(out.logical_view()), bits(ref.grid.logical_view()))
    finally:
        product.wg_session_destroy(s)


def test_swe_nonpositive_depth_fails_loudly(product):
    cfg = swe_cfg(65, (2, 2), 3, 5e-4, 0.01)
    g0 = api.initial_state(cfg, lib=product)
    g0.logical_view()[1, 0, 5, 5] = 0.0  # patch 1, component h
    s = _session(product, cfg)
    try:
        st = product.wg_session_upload(s, abi.dptr(g0.data))
        if st == 0:
            st = product.wg_session_sync(s)
        assert st == 5  # WG_DOMAIN
    finally:
        product.wg_session_destroy(s)


@pytest.mark.parametrize("scheme", ["transport", "lbm", "swe"])
def test_many_patches_per_cta(product, oracle_sq, monkeypatch, scheme):
    """Persistent CTAs looping over many patches (the large-grid regime: C2-C5
    put 4-40 patches on every CTA): a launch grid of a few CTAs must give the
    same bits as one CTA per patch."""
    monkeypatch.setenv("WG_GRID_WAVES", "0.004")  # ~1-2 CTAs on 148 SMs
    if scheme == "swe":
        cfg = swe_cfg(257, (4, 4), 4, 5e-4, 0.004)
    elif scheme == "lbm":
        cfg = api.RunConfig(scheme="lbm", nx=257, splits=(8, 8), levels=4, lbm_steps=4,
                            spec=api.ThresholdSpec("capped", 1e-3))
    else:
        cfg = api.RunConfig(scheme="transport", nx=257, splits=(8, 8), levels=4,
                            spec=api.ThresholdSpec("capped", 1e-3), compute_l2=False)
        cfg.t_end = 6 * cfg.cfl / 256 / 0.9
    compare_runs(api.run(cfg, lib=product), api.run(cfg, lib=oracle_sq))
