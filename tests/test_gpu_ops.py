"""Per-op parity of the sm_100a kernels against the C oracle (bit-exact),
through the C ABI.  Mirrors the reference's unit suites (test_wavelet.cpp,
test_threshold.cpp, test_codec.cpp, test_patchgrid.cpp, test_solver.cpp)."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2302_09883_b200 import abi, api

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.mark.parametrize(
    "dims,levels",
    [((9,), 3), ((129,), 7), ((17, 17), 2), ((33, 33), 4), ((65, 65), 4), ((65, 65), 6), ((17, 33), 3),
     ((9, 9, 9), 2), ((17, 17, 17), 3), ((5, 3), 1), ((1025,), 10), ((2, 2), 0)],
)
def test_dwt_idwt_bit_exact(product, oracle, dims, levels):
    rng = np.random.default_rng(hash(dims) % 2**32)
    x = rng.uniform(-1, 1, size=dims)
    c_dev = api.dwt_nd(x, levels, lib=product)
    c_ref = api.dwt_nd(x, levels, lib=oracle)
    assert np.array_equal(bits(c_dev), bits(c_ref))
    r_dev = api.idwt_nd(c_dev, levels, lib=product)
    r_ref = api.idwt_nd(c_ref, levels, lib=oracle)
    assert np.array_equal(bits(r_dev), bits(r_ref))
    assert np.max(np.abs(r_dev - x)) <= 1e-14  # test_wavelet.cpp:165-191


def test_invalid_plans_rejected(product):
    with pytest.raises(abi.InvalidArgument):
        api.dwt_nd(np.zeros((9, 9)), 4, lib=product)  # test_wavelet.cpp:138-139
    with pytest.raises(abi.InvalidArgument):
        api.dwt_nd(np.zeros((10,)), 1, lib=product)


def test_impulse_and_ramp_kat(product):
    s = np.zeros(9)
    s[0] = 1.0
    c = api.dwt_nd(s, 1, lib=product)  # corner layout: coarse 0..4, details 5..8
    inter = np.empty(9)
    inter[0::2], inter[1::2] = c[:5], c[5:]
    assert list(inter) == [1, -0.5, -0.25, 0, 0, 0, 0, 0, 0]  # test_wavelet.cpp:69-75
    ramp = np.arange(5.0)
    c = api.dwt_nd(ramp, 1, lib=product)
    assert list(c) == [0, 2, 4, 0, 0]  # test_wavelet.cpp:61-67


@pytest.mark.parametrize("mode", ["constant", "accumulation", "capped"])
@pytest.mark.parametrize("dims,levels,c", [((33, 33), 3, 0.05), ((65, 65), 4, 1e-3), ((17, 17, 17), 3, 0.1),
                                           ((9,), 2, 0.3), ((65, 65), 6, 0.5)])
def test_threshold_bit_exact(product, oracle, mode, dims, levels, c):
    rng = np.random.default_rng(7)
    x = rng.uniform(-1, 1, size=dims) * rng.uniform(0, 1, size=dims) ** 4
    x.flat[::7] = 0.0
    x.flat[1::11] = -0.0
    spec = api.ThresholdSpec(mode, c, 2.0)
    a, b = x.copy(), x.copy()
    za = api.apply_threshold(a, levels, spec, lib=product)
    zb = api.apply_threshold(b, levels, spec, lib=oracle)
    assert za == zb
    assert np.array_equal(bits(a), bits(b))


def test_threshold_strict_comparison(product):
    cs = np.zeros(9)
    cs[5] = 0.2
    cs[6] = np.nextafter(0.2, 0.0)  # test_threshold.cpp:47-55
    assert api.apply_threshold(cs, 1, api.ThresholdSpec("constant", 0.2), lib=product) == 1
    assert cs[5] == 0.2 and cs[6] == 0.0
    with pytest.raises(abi.InvalidArgument):
        api.apply_threshold(np.zeros(9), 1, api.ThresholdSpec("capped", -1.0), lib=product)


def test_samples_never_modified(product):
    rng = np.random.default_rng(5)
    cs = rng.uniform(-1, 1, (33, 33))
    before = cs.copy()
    api.apply_threshold(cs, 3, api.ThresholdSpec("constant", np.inf), lib=product)
    nb = (32 >> 3) + 1
    assert np.array_equal(cs[:nb, :nb], before[:nb, :nb])
    mask = np.ones_like(cs, bool)
    mask[:nb, :nb] = False
    assert np.all(cs[mask] == 0.0)


@pytest.mark.parametrize("rows,cols,density", [(3, 3, 0.0), (1, 1, 1.0), (13, 17, 0.3), (65, 65, 0.05),
                                               (200, 37, 0.5), (1, 100, 0.9)])
def test_csr_roundtrip_bit_exact(product, oracle, rows, cols, density):
    rng = np.random.default_rng(rows * 1000 + cols)
    m = np.where(rng.uniform(size=(rows, cols)) < density, rng.uniform(-5, 5, (rows, cols)), 0.0)
    m.flat[::5] *= -0.0 if density < 1 else 1.0
    a = api.csr_encode(m, rows, cols, lib=product)
    b = api.csr_encode(m, rows, cols, lib=oracle)
    assert np.array_equal(bits(a.v), bits(b.v))
    assert np.array_equal(a.col, b.col) and np.array_equal(a.row, b.row)
    assert a.byte_size() == 12 * a.nnz() + 4 * (rows + 1)  # codec.hpp:33
    d = api.csr_decode(a, lib=product)
    assert np.array_equal(d, m.reshape(-1))


def test_csr_corrupt_rejected(product):
    b = api.csr_encode(np.array([1.0, 0, 0, 1]), 2, 2, lib=product)
    bad = api.CsrBlock(b.v, b.col.copy(), b.row, 2, 2)
    bad.col[0] = 5  # test_codec.cpp:59-69
    with pytest.raises(abi.CorruptStreamError):
        api.csr_decode(bad, lib=product)
    bad = api.CsrBlock(b.v, b.col, b.row.copy(), 2, 2)
    bad.row[-1] = 9
    with pytest.raises(abi.CorruptStreamError):
        api.csr_decode(bad, lib=product)


def test_ghost_sync_kats(product):
    g = api.decompose((9,), (2,), 1, lib=product)
    api.fill(g, 0, lambda i: float(i[0]))
    api.sync_ghosts(g, lib=product)
    left, right = g.data[0, 0], g.data[1, 0]
    assert left[6] == 5.0 and right[0] == 3.0 and left[0] == 7.0 and right[6] == 1.0  # test_patchgrid.cpp:45-69
    g = api.decompose((9, 9), (2, 2), 1, lib=product)
    api.fill(g, 0, lambda i: float(i[0] * 100 + i[1]))
    api.sync_ghosts(g, lib=product)
    assert g.data[0, 0, 6, 6] == 505.0 and g.data[0, 0, 0, 0] == 707.0  # test_patchgrid.cpp:93-104
    g = api.decompose((5,), (1,), 1, periodic=False, lib=product)
    api.fill(g, 0, lambda i: float(i[0] ** 2))
    api.sync_ghosts(g, lib=product)
    assert g.data[0, 0, 0] == g.data[0, 0, 1] and g.data[0, 0, 6] == g.data[0, 0, 5]


@pytest.mark.parametrize("gd,sp,m,per", [((33, 33), (2, 2), 1, True), ((65, 65), (4, 2), 3, True),
                                         ((17, 17, 9), (2, 1, 2), 2, True), ((33, 33), (2, 4), 9, False)])
def test_sync_ghosts_bit_exact(product, oracle, gd, sp, m, per):
    g1 = api.PatchGrid(gd, sp, m, per)
    rng = np.random.default_rng(3)
    g1.data[...] = rng.uniform(size=g1.data.shape)
    g2 = api.PatchGrid(gd, sp, m, per, data=g1.data.copy())
    api.sync_ghosts(g1, lib=product)
    api.sync_ghosts(g2, lib=oracle)
    assert np.array_equal(bits(g1.data), bits(g2.data))


def test_global_mass(product, oracle):
    g = api.decompose((129, 129), (2, 2), 1, lib=product)
    g.logical_view()[...] = 1.0
    assert abs(api.global_mass(g, 0, lib=product) - 128.0 * 128.0) <= 1e-13 * 128 * 128  # test_patchgrid.cpp:128-133
    rng = np.random.default_rng(11)
    g.data[...] = rng.uniform(size=g.data.shape)
    a, b = api.global_mass(g, 0, lib=product), api.global_mass(g, 0, lib=oracle)
    assert abs(a - b) <= 1e-12 * abs(b)


def _random_state(gd, sp, m, seed, lo=1.0, hi=2.0):
    g = api.PatchGrid(gd, sp, m, True)
    rng = np.random.default_rng(seed)
    g.data[...] = rng.uniform(lo, hi, size=g.data.shape)
    return g


@pytest.mark.parametrize("alpha,beta", [(0.9, 0.9), (1.0, 0.0), (-0.4, 0.7), (0.0, -1.3)])
def test_fv_transport_bit_exact(product, oracle, alpha, beta):
    cur = _random_state((33, 33), (2, 2), 1, 1)
    api.sync_ghosts(cur, lib=oracle)
    n1 = api.PatchGrid((33, 33), (2, 2), 1, True, data=np.zeros_like(cur.data))
    n2 = api.PatchGrid((33, 33), (2, 2), 1, True, data=np.zeros_like(cur.data))
    api.fv_step(cur, n1, "transport", 0.01, 1 / 32, alpha, beta, lib=product)
    api.fv_step(cur, n2, "transport", 0.01, 1 / 32, alpha, beta, lib=oracle)
    assert np.array_equal(bits(n1.data), bits(n2.data))


def test_fv_swe_bit_exact(product, oracle):
    cur = _random_state((33, 33), (2, 2), 3, 2, 0.5, 1.5)
    cur.data[:, 1:] -= 1.0  # momenta around 0
    api.sync_ghosts(cur, lib=oracle)
    n1 = api.PatchGrid((33, 33), (2, 2), 3, True, data=np.zeros_like(cur.data))
    n2 = api.PatchGrid((33, 33), (2, 2), 3, True, data=np.zeros_like(cur.data))
    api.fv_step(cur, n1, "swe", 1e-3, 1 / 32, lib=product)
    api.fv_step(cur, n2, "swe", 1e-3, 1 / 32, lib=oracle)
    assert np.array_equal(bits(n1.data), bits(n2.data))
    bad = _random_state((17, 17), (1, 1), 3, 3)
    bad.data[0, 0, 5, 5] = -1.0
    with pytest.raises(abi.DomainError):
        api.fv_step(bad, api.PatchGrid((17, 17), (1, 1), 3, True), "swe", 1e-3, 1 / 16, lib=product)


def test_lbm_step_bit_exact(product, oracle):
    cur = _random_state((33, 33), (2, 2), 9, 4, 0.01, 0.2)
    api.sync_ghosts(cur, lib=oracle)
    n1 = api.PatchGrid((33, 33), (2, 2), 9, True, data=np.zeros_like(cur.data))
    n2 = api.PatchGrid((33, 33), (2, 2), 9, True, data=np.zeros_like(cur.data))
    api.lbm_step(cur, n1, 0.6, lib=product)
    api.lbm_step(cur, n2, 0.6, lib=oracle)
    assert np.array_equal(bits(n1.data), bits(n2.data))


def test_demo_discontinuous_golden(product):
    """pipeline.hpp:417-460 / PAPER.md:481 on the device, against the
    reference-generated golden hashes (tests/golden/kat.json)."""
    import hashlib
    import json

    from tests.conftest import GOLDEN
    from tests.golden.make_golden import demo_field

    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    kat = json.loads((GOLDEN / "kat.json").read_text())["demo"]
    f = demo_field()
    cs = api.dwt_nd(f, 6, lib=product)
    assert api.apply_threshold(cs, 6, api.ThresholdSpec("constant", 0.2), lib=product) == kat["zeroed"]
    assert sha(cs) == kat["coeff_sha256"] and int(np.count_nonzero(cs)) == 481
    assert sha(api.idwt_nd(cs, 6, lib=product)) == kat["recon_sha256"]
    blk = api.csr_encode(cs, 129, 129, lib=product)
    assert sha(blk.v) == kat["csr_v_sha256"] and sha(blk.col) == kat["csr_col_sha256"]
    assert sha(blk.row) == kat["csr_row_sha256"]


@pytest.mark.parametrize("name", ["small_transport", "small_lbm"])
def test_run_goldens_on_device(product, name):
    import hashlib
    import json

    from tests.conftest import GOLDEN

    gold = json.loads((GOLDEN / f"{name}.json").read_text())
    c = gold["config"]
    cfg = api.RunConfig(scheme=c["scheme"], nx=c["nx"], splits=tuple(c["splits"]), levels=c["levels"],
                        t_end=c["t_end"], lbm_steps=c["lbm_steps"], compute_l2=False,
                        spec=api.ThresholdSpec(c["spec"]["mode"], c["spec"]["c"], c["spec"]["alpha"]))
    r = api.run(cfg, lib=product)
    assert len(r.rows) == gold["steps"]
    for row, g in zip(r.rows, gold["rows"]):
        assert (row["nnz"], row["zeroed"], row["compressed_bytes"]) == (g["nnz"], g["zeroed"], g["compressed_bytes"])
    assert hashlib.sha256(np.ascontiguousarray(r.grid.logical_view()).tobytes()).hexdigest() == gold["state_sha256"]
