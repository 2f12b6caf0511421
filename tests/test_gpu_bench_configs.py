"""Device parity at the bench configurations themselves (BASELINE.json
configs[1] = C2 and configs[2] = C3, SURVEY §8 config map), not just their
patch shapes: the product's run() against the C oracle's run()
(pipeline.hpp:129-305 restated) — state and integer metrics bit-exact, mass
within 1e-12 — plus the stored CSR blocks of sampled patches against
csr_encode of the oracle's thresholded coefficients (codec.hpp:37-60)."""
from __future__ import annotations

import ctypes as C
import math

import numpy as np
import pytest

from paper_2302_09883_b200 import abi, api

from .test_gpu_session import _session, bits, compare_runs, lbm_cfg
from .test_gpu_swe import swe_cfg

pytestmark = pytest.mark.gpu

C2 = dict(nx=1025, splits=(16, 16), levels=4, c=1e-3)        # D2Q9 1024^2, 64^2-cell patches
C3 = dict(nx=4097, splits=(64, 64), levels=4, c=5e-4)        # SWE dam break 4096^2


def test_c2_exact_config_parity(product, oracle):
    """C2 exactly: 1025^2 points, 16 x 16 patches of 65^2, L = 4, capped
    1e-3, 20 steps — state, nnz/zeroed/bytes of every row, mass."""
    cfg = lbm_cfg(C2["nx"], C2["splits"], C2["levels"], C2["c"], 20)
    compare_runs(api.run(cfg, lib=product), api.run(cfg, lib=oracle))


def test_c2_csr_blocks_sampled(product, oracle):
    """The device store after step 20 of C2 holds, for sampled patches and
    every population, exactly csr_encode(apply_threshold(dwt_nd(.))) of the
    oracle's collided state of step 20."""
    steps = 20
    g = api.run(lbm_cfg(C2["nx"], C2["splits"], C2["levels"], C2["c"], steps - 1), lib=oracle).grid
    api.sync_ghosts(g, lib=oracle)
    nxt = api.PatchGrid(g.global_dims, g.splits, 9, True, data=g.data.copy())
    api.lbm_step(g, nxt, 0.6, lib=oracle)
    cfg = lbm_cfg(C2["nx"], C2["splits"], C2["levels"], C2["c"], steps)
    s = _session(product, cfg)
    try:
        g0 = api.initial_state(cfg, lib=oracle)
        product.check(product.wg_session_upload(s, abi.dptr(g0.data)))
        for _ in range(steps):
            product.check(product.wg_session_step(s, 1.0))
        product.check(product.wg_session_sync(s))
        for p in (0, 1, 17, 100, 255):
            for q in range(9):
                blk = np.ascontiguousarray(nxt.data[p, q, 1:-1, 1:-1])
                cs = api.dwt_nd(blk, C2["levels"], lib=oracle)
                api.apply_threshold(cs, C2["levels"], cfg.spec, lib=oracle)
                want = api.csr_encode(cs, 65, 65, lib=oracle)
                nnz, raw = abi.u64(), abi.i32()
                product.check(product.wg_session_patch_csr(s, p, q, None, None, None, C.byref(nnz), C.byref(raw)))
                assert raw.value == 0 and nnz.value == want.nnz(), (p, q)
                v = np.empty(nnz.value)
                col = np.empty(nnz.value, np.uint32)
                row = np.empty(66, np.uint32)
                product.check(product.wg_session_patch_csr(
                    s, p, q, abi.dptr(v), col.ctypes.data_as(C.POINTER(abi.u32)),
                    row.ctypes.data_as(C.POINTER(abi.u32)), C.byref(nnz), C.byref(raw)))
                assert np.array_equal(bits(v), bits(want.v)), (p, q)
                assert np.array_equal(col, want.col) and np.array_equal(row, want.row), (p, q)
    finally:
        product.wg_session_destroy(s)


def test_c3_exact_config_parity(product, oracle_sq):
    """C3 exactly: SWE dam break, 4097^2 points, 64 x 64 patches of 65^2,
    L = 4, constant 5e-4, >= 5 steps (t_end 1.5e-4 s) — bit-exact against
    the restatement with the Newton start squared by multiplication (the
    device's arithmetic, tests/test_gpu_swe.py)."""
    cfg = swe_cfg(C3["nx"], C3["splits"], C3["levels"], C3["c"], 1.5e-4, "constant")
    a = api.run(cfg, lib=product)
    b = api.run(cfg, lib=oracle_sq)
    assert len(a.rows) >= 5
    # mass: 16.8 M cells summed in different orders (the oracle serially,
    # the device as a tree) differ by ~1e-12 relative; both are checked
    # against the exactly rounded trapezoid sum of the final state
    compare_runs(a, b, mass_rtol=1e-11)
    g = a.grid
    w = np.ones(65)
    w[0] = w[-1] = 0.5
    h = g.data[:, 0, 1:-1, 1:-1] * np.outer(w, w)
    exact = math.fsum(h.ravel())
    assert abs(a.rows[-1]["global_mass"] - exact) <= 1e-13 * exact
    assert abs(b.rows[-1]["global_mass"] - exact) <= 1e-11 * exact
    m0 = a.rows[0]["global_mass"]
    assert all(abs(r["global_mass"] - m0) <= 1e-12 * m0 for r in a.rows)


@pytest.mark.parametrize("stream_rows", [None, 1, 3])
def test_budget_streamed_first_step(product, oracle, monkeypatch, stream_rows):
    """Budget mode with a host initial state (the C4 path): the store budget
    is below the raw state, so run() streams the host grid into step 1
    (wg_session_step_host, in patch-row chunks) and the raw state never
    enters the store — results identical to the oracle's run() bit for bit,
    for one chunk and for several (WG_STREAM_ROWS)."""
    if stream_rows:
        monkeypatch.setenv("WG_STREAM_ROWS", str(stream_rows))
    cfg = lbm_cfg(257, (4, 4), 4, 1e-3, 6)
    raw = 16 * 9 * 33808  # the raw store of 16 patches x 9 populations
    cfg.store_budget_bytes = 2 * 1024 * 1024  # pools of 1 MiB: a quarter of the raw state
    assert cfg.store_budget_bytes // 2 < raw
    compare_runs(api.run(cfg, lib=product), api.run(cfg, lib=oracle))


def test_step_host_equals_upload(product):
    """wg_session_step_host == wg_session_upload + wg_session_step (state and
    rows), chunked download included."""
    cfg = lbm_cfg(257, (4, 4), 4, 1e-3, 5)
    g0 = api.initial_state(cfg, lib=product).data.reshape(-1).copy()

    def go(streamed):
        s = _session(product, cfg)
        try:
            if streamed:
                product.check(product.wg_session_step_host(s, abi.dptr(g0), 1.0))
            else:
                product.check(product.wg_session_upload(s, abi.dptr(g0)))
                product.check(product.wg_session_step(s, 1.0))
            for _ in range(4):
                product.check(product.wg_session_step(s, 1.0))
            out = np.zeros_like(g0)
            product.check(product.wg_session_download(s, abi.dptr(out)))
            rows = (abi.MetricsRowC * 5)()
            n = abi.u64()
            product.check(product.wg_session_metrics(s, rows, 5, C.byref(n)))
            return out, [(r.step, r.nnz, r.zeroed, r.compressed_bytes, r.global_mass) for r in rows[: n.value]]
        finally:
            product.wg_session_destroy(s)

    a, ra = go(True)
    b, rb = go(False)
    assert ra == rb and len(ra) == 5
    assert np.array_equal(bits(a), bits(b))


@pytest.mark.parametrize("c", [1e-12, 1e-7])
def test_c2_grid_tiny_threshold(product, oracle, c):
    """The C2 grid at thresholds that zero almost nothing: every patch's
    blocks are nearly dense CSR (up to 1.5x the raw block), or raw by the
    skip rule — the default store pools (sized for the dense-CSR worst case)
    never overflow, and the run equals the reference's bit for bit."""
    cfg = lbm_cfg(C2["nx"], C2["splits"], C2["levels"], c, 3)
    compare_runs(api.run(cfg, lib=product), api.run(cfg, lib=oracle))


def test_c4_full_size_streamed_equals_uploaded(product):
    """C4 at its full size (16384^2, 256 x 256 patches of 65^2, L = 4, capped
    1e-3) with the host initial state: the bench path (store budget 8 GiB,
    the raw state streamed into step 1, wg_session_step_host) against the
    plain path (no budget: the raw state uploaded into the store first) —
    two different code paths, the same result: every metrics row equal
    (nnz, zeroed, bytes; mass to 1e-13), the stored CSR blocks of sampled
    patches (all 9 populations) bitwise equal; and the size-independent
    properties: mass conserved to round-off, every block at the L = 4 floor
    (25 samples: 564 bytes)."""
    cfg = lbm_cfg(16385, (256, 256), 4, 1e-3, 4)
    g0 = api.initial_state(cfg, lib=product).data.reshape(-1)
    steps = 4
    samples = [0, 255, 256 * 128 + 77, 65535 - 256, 65535]

    def block(s, p, q):
        nnz, raw = abi.u64(), abi.i32()
        product.check(product.wg_session_patch_csr(s, p, q, None, None, None, C.byref(nnz), C.byref(raw)))
        v = np.empty(max(nnz.value, 1))
        col = np.empty(max(nnz.value, 1), np.uint32)
        row = np.empty(66, np.uint32)
        product.check(product.wg_session_patch_csr(
            s, p, q, abi.dptr(v), col.ctypes.data_as(C.POINTER(abi.u32)),
            row.ctypes.data_as(C.POINTER(abi.u32)), C.byref(nnz), C.byref(raw)))
        return raw.value, bits(v[: nnz.value]).tobytes(), col[: nnz.value].tobytes(), row.tobytes()

    def go(budget):
        cfg.store_budget_bytes = budget
        s = _session(product, cfg)
        try:
            if budget:
                product.check(product.wg_session_step_host(s, abi.dptr(g0), 1.0))
            else:
                product.check(product.wg_session_upload(s, abi.dptr(g0)))
                product.check(product.wg_session_step(s, 1.0))
            for _ in range(steps - 1):
                product.check(product.wg_session_step(s, 1.0))
            rows = (abi.MetricsRowC * steps)()
            n = abi.u64()
            product.check(product.wg_session_metrics(s, rows, steps, C.byref(n)))
            r = [(x.step, x.nnz, x.zeroed, x.compressed_bytes, x.dense_bytes, x.global_mass) for x in rows[: n.value]]
            blocks = {(p, q): block(s, p, q) for p in samples for q in range(9)}
            return r, blocks
        finally:
            product.wg_session_destroy(s)

    ra, ba = go(8 << 30)
    rb, bb = go(0)
    assert len(ra) == steps and [x[:5] for x in ra] == [x[:5] for x in rb]
    # masses: the streamed step 1 sums its patch-row chunks' partials in
    # another (fixed) order than one launch does
    assert all(abs(x[5] - y[5]) <= 1e-13 * abs(y[5]) for x, y in zip(ra, rb))
    assert ba == bb
    npatch = 256 * 256
    m0 = ra[0][5]
    for step, nnz, zeroed, cb, db, mass in ra:
        assert nnz == npatch * 9 * 25 and cb == npatch * 9 * 564 and db == npatch * 9 * 65 * 65 * 8
        assert abs(mass - m0) <= 1e-12 * abs(m0)
