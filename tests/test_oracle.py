"""CPU: pin the C restatement (oracle/wg_oracle.c) to the reference.

Against the committed golden vectors (generated from the reference headers
themselves, tests/golden/make_golden.py) and, where oracle/_ref was built in
this container, directly against the compiled reference on seeded inputs.
Known-answer tests follow the reference's own suites (file:line cited)."""
from __future__ import annotations

import hashlib
import json
import math

import numpy as np
import pytest

from paper_2302_09883_b200 import abi, api

from .conftest import GOLDEN


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def hexd(x):
    return np.float64(x).view(np.uint64).item().to_bytes(8, "big").hex()


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---- known answers (reference test suites) -----------------------------------


def test_impulse_ramp_and_analysis_matrix(oracle):
    s = np.zeros(9)
    s[0] = 1.0
    c = api.dwt_nd(s, 1, lib=oracle)
    inter = np.empty(9)
    inter[0::2], inter[1::2] = c[:5], c[5:]
    assert list(inter) == [1, -0.5, -0.25, 0, 0, 0, 0, 0, 0]  # test_wavelet.cpp:69-75
    assert list(api.dwt_nd(np.arange(5.0), 1, lib=oracle)) == [0, 2, 4, 0, 0]  # :61-67
    # analysis matrix j=3 (test_wavelet.cpp:14-23, 77-82): columns are impulse responses
    A9 = np.array([[8, 0, 0, 0, 0, 0, 0, 0, 0], [-4, 8, -4, 0, 0, 0, 0, 0, 0], [-2, 4, 5, 2, -1, 0, 0, 0, 0],
                   [0, 0, -4, 8, -4, 0, 0, 0, 0], [0, 0, -1, 2, 6, 2, -1, 0, 0], [0, 0, 0, 0, -4, 8, -4, 0, 0],
                   [0, 0, 0, 0, -1, 2, 5, 4, -2], [0, 0, 0, 0, 0, 0, -4, 8, -4], [0, 0, 0, 0, 0, 0, 0, 0, 8]]) / 8.0
    for r in range(9):
        e = np.zeros(9)
        e[r] = 1.0
        c = api.dwt_nd(e, 1, lib=oracle)
        col = np.empty(9)
        col[0::2], col[1::2] = c[:5], c[5:]
        assert np.array_equal(col, A9[:, r])


def test_band_threshold_laws(oracle):
    assert api.band_threshold([3, 1], api.ThresholdSpec("constant", 0.01), lib=oracle) == 0.01
    assert api.band_threshold([3, 1], api.ThresholdSpec("capped", 0.01, 2.0), lib=oracle) == pytest.approx(0.08)
    assert api.band_threshold([3, 1], api.ThresholdSpec("accumulation", 0.01, 2.0), lib=oracle) == pytest.approx(0.16)
    assert api.band_threshold([0, 0], api.ThresholdSpec("capped", 0.01, 2.0), lib=oracle) == 0.01


def test_threshold_strictness_and_samples(oracle):
    cs = np.zeros(9)
    cs[5] = 0.2
    cs[6] = np.nextafter(0.2, 0.0)
    assert api.apply_threshold(cs, 1, api.ThresholdSpec("constant", 0.2), lib=oracle) == 1
    assert cs[5] == 0.2 and cs[6] == 0.0  # test_threshold.cpp:47-55
    with pytest.raises(abi.InvalidArgument):
        api.apply_threshold(np.zeros(9), 1, api.ThresholdSpec("capped", -1.0), lib=oracle)


def test_csr_kats(oracle):
    z = api.csr_encode(np.zeros(9), 3, 3, lib=oracle)
    assert z.nnz() == 0 and list(z.row) == [0, 0, 0, 0]  # test_codec.cpp:21-28
    eye = api.csr_encode(np.eye(3).reshape(-1), 3, 3, lib=oracle)
    assert list(eye.col) == [0, 1, 2] and list(eye.row) == [0, 1, 2, 3]
    blk = api.csr_encode(np.zeros(65 * 65), 65, 65, lib=oracle)
    assert blk.byte_size() == 4 * 66  # test_codec.cpp:163-169
    bad = api.CsrBlock(eye.v, eye.col.copy(), eye.row, 3, 3)
    bad.col[0] = 5
    with pytest.raises(abi.CorruptStreamError):
        api.csr_decode(bad, lib=oracle)


def test_ghost_and_mass_kats(oracle):
    g = api.decompose((9,), (2,), 1, lib=oracle)
    api.fill(g, 0, lambda i: float(i[0]))
    api.sync_ghosts(g, lib=oracle)
    assert g.data[0, 0, 6] == 5.0 and g.data[1, 0, 0] == 3.0  # test_patchgrid.cpp:45-69
    assert g.data[0, 0, 0] == 7.0 and g.data[1, 0, 6] == 1.0
    g = api.decompose((9, 9), (2, 2), 1, lib=oracle)
    api.fill(g, 0, lambda i: float(i[0] * 100 + i[1]))
    api.sync_ghosts(g, lib=oracle)
    assert g.data[0, 0, 6, 6] == 505.0 and g.data[0, 0, 0, 0] == 707.0  # :93-104
    g = api.decompose((129, 129), (2, 2), 1, lib=oracle)
    g.logical_view()[...] = 1.0
    assert api.global_mass(g, 0, lib=oracle) == pytest.approx(128.0 * 128.0, rel=1e-13)  # :128-133
    with pytest.raises(abi.InvalidArgument):
        api.decompose((13,), (2,), 1, lib=oracle)  # 7 is not 2^k+1


def test_demo_discontinuous_481(oracle):
    """pipeline.hpp:417-460: 481 of 16641 coefficients survive."""
    from tests.golden.make_golden import demo_field

    kat = json.loads((GOLDEN / "kat.json").read_text())["demo"]
    f = demo_field()
    assert sha(f) == kat["field_sha256"]  # glibc exp/sin through math.*
    cs = api.dwt_nd(f, 6, lib=oracle)
    z = api.apply_threshold(cs, 6, api.ThresholdSpec("constant", 0.2), lib=oracle)
    assert z == kat["zeroed"]
    assert sha(cs) == kat["coeff_sha256"]  # thresholded coefficients
    assert int(np.count_nonzero(cs)) == kat["nonzeros"] == 481
    assert sha(api.idwt_nd(cs, 6, lib=oracle)) == kat["recon_sha256"]
    blk = api.csr_encode(cs, 129, 129, lib=oracle)
    assert sha(blk.v) == kat["csr_v_sha256"] and sha(blk.col) == kat["csr_col_sha256"]
    assert sha(blk.row) == kat["csr_row_sha256"]


def test_random33_golden(oracle):
    kat = json.loads((GOLDEN / "kat.json").read_text())["random33_L4"]
    x = np.random.default_rng(kat["seed"]).uniform(-1, 1, (33, 33))
    assert sha(x) == kat["input_sha256"]
    c = api.dwt_nd(x, 4, lib=oracle)
    assert sha(c) == kat["coeff_sha256"]
    assert sha(api.idwt_nd(c, 4, lib=oracle)) == kat["recon_sha256"]
    assert api.apply_threshold(c, 4, api.ThresholdSpec("capped", 0.05), lib=oracle) == kat["capped_0.05_zeroed"]
    assert sha(c) == kat["capped_0.05_sha256"]


# ---- run() goldens (generated by the reference) ------------------------------


def _check_run_golden(oracle, name, cfg):
    gold = json.loads((GOLDEN / f"{name}.json").read_text())
    r = api.run(cfg, lib=oracle)
    assert len(r.rows) == gold["steps"]
    for row, g in zip(r.rows, gold["rows"]):
        for k in ("step", "dense_bytes", "compressed_bytes", "nnz", "zeroed"):
            assert row[k] == g[k], (k, row, g)
        for k in ("time", "ratio", "global_mass", "l2"):
            assert hexd(row[k]) == g[k], (k, row[k])
    assert hexd(r.summary["avg_ratio"]) == gold["avg_ratio_hex"]
    assert sha(r.grid.logical_view()) == gold["state_sha256"]


def test_small_transport_golden(oracle):
    _check_run_golden(oracle, "small_transport",
                      api.RunConfig(scheme="transport", nx=33, splits=(2, 2), levels=3, t_end=0.05,
                                    spec=api.ThresholdSpec("capped", 0.01)))


def test_small_swe_golden(oracle):
    _check_run_golden(oracle, "small_swe",
                      api.RunConfig(scheme="swe", nx=33, splits=(2, 2), levels=3, t_end=0.05,
                                    spec=api.ThresholdSpec("constant", 0.0005)))


def test_small_lbm_golden(oracle):
    _check_run_golden(oracle, "small_lbm",
                      api.RunConfig(scheme="lbm", nx=129, splits=(4, 4), levels=4, lbm_steps=20,
                                    spec=api.ThresholdSpec("capped", 1e-3)))


@pytest.mark.slow
def test_c1_golden(oracle):
    """C1: 256^2 cells, 8x8 patches of 33^2, level 4, capped 1e-3, 100 steps
    (SURVEY §8c probe goldens: nnz 800, zeroed 60105, 18304 B, l2 3.515e-5)."""
    gold = json.loads((GOLDEN / "c1_transport.json").read_text())
    assert gold["final"]["nnz"] == 800 and gold["final"]["zeroed"] == 60105
    _check_run_golden(oracle, "c1_transport",
                      api.RunConfig(scheme="transport", nx=257, splits=(8, 8), levels=4, t_end=100 / 512,
                                    spec=api.ThresholdSpec("capped", 1e-3)))


# ---- direct comparison with the compiled reference (build container only) ----


@pytest.mark.parametrize("dims,levels", [((33, 33), 4), ((65, 65), 5), ((17, 33), 3), ((9, 9, 9), 2),
                                         ((129,), 7), ((5,), 2), ((17, 17, 17), 3)])
def test_transforms_vs_reference(oracle, reference, dims, levels):
    x = np.random.default_rng(len(dims) * 7 + levels).uniform(-1, 1, dims)
    for f in (api.dwt_nd, api.idwt_nd):
        assert np.array_equal(bits(f(x, levels, lib=oracle)), bits(f(x, levels, lib=reference)))
    for mode in ("constant", "accumulation", "capped"):
        a, b = api.dwt_nd(x, levels, lib=oracle), api.dwt_nd(x, levels, lib=reference)
        spec = api.ThresholdSpec(mode, 0.07, 1.7)
        assert api.apply_threshold(a, levels, spec, lib=oracle) == api.apply_threshold(b, levels, spec, lib=reference)
        assert np.array_equal(bits(a), bits(b))


def test_grid_ops_vs_reference(oracle, reference):
    rng = np.random.default_rng(5)
    for gd, sp, m, per in [((17, 17), (2, 2), 1, True), ((33, 33), (2, 4), 3, False), ((9, 17, 9), (2, 2, 1), 2, True)]:
        a = api.PatchGrid(gd, sp, m, per)
        a.data[...] = rng.uniform(size=a.data.shape)
        b = api.PatchGrid(gd, sp, m, per, data=a.data.copy())
        api.sync_ghosts(a, lib=oracle)
        api.sync_ghosts(b, lib=reference)
        assert np.array_equal(bits(a.data), bits(b.data))
        for c in range(m):
            assert hexd(api.global_mass(a, c, lib=oracle)) == hexd(api.global_mass(b, c, lib=reference))
    cur = api.PatchGrid((33, 33), (2, 2), 3, True)
    cur.data[...] = rng.uniform(0.5, 1.5, cur.data.shape)
    cur.data[:, 1:] -= 1.0
    n1, n2 = api.PatchGrid((33, 33), (2, 2), 3, True), api.PatchGrid((33, 33), (2, 2), 3, True)
    api.fv_step(cur, n1, "swe", 1e-3, 1 / 32, lib=oracle)
    api.fv_step(cur, n2, "swe", 1e-3, 1 / 32, lib=reference)
    assert np.array_equal(bits(n1.data), bits(n2.data))


@pytest.mark.parametrize("cfg", [
    api.RunConfig(scheme="transport", nx=65, splits=(2, 2), levels=4, t_end=0.03,
                  spec=api.ThresholdSpec("accumulation", 0.004)),
    api.RunConfig(scheme="transport", nx=33, splits=(2, 2), levels=3, t_end=0.05, spec=api.ThresholdSpec("capped", 0.0),
                  strict=True),
    api.RunConfig(scheme="swe", nx=65, splits=(2, 2), levels=4, t_end=0.01, cfl=0.2,
                  spec=api.ThresholdSpec("constant", 5e-4)),
    api.RunConfig(scheme="lbm", nx=65, splits=(2, 2), levels=4, lbm_steps=8, spec=api.ThresholdSpec("capped", 1e-4)),
], ids=["transport-accum", "transport-c0-strict", "swe", "lbm"])
def test_run_vs_reference(oracle, reference, cfg):
    a, b = api.run(cfg, lib=oracle), api.run(cfg, lib=reference)
    assert [{k: r[k] for k in r} for r in a.rows] == [{k: r[k] for k in r} for r in b.rows]
    assert np.array_equal(bits(a.grid.logical_view()), bits(b.grid.logical_view()))


def test_error_types_vs_reference(oracle, reference):
    for lib in (oracle, reference):
        with pytest.raises(abi.InvalidArgument):
            api.dwt_nd(np.zeros((9, 9)), 4, lib=lib)  # WaveletPlan::validate
        with pytest.raises(abi.InvalidArgument):
            api.run(api.RunConfig(cfl=1.5), lib=lib)  # SimConfig::validate
        bad = api.PatchGrid((17, 17), (1, 1), 3, True)
        bad.data[0, 0, 5, 5] = -1.0
        with pytest.raises(abi.DomainError):
            api.fv_step(bad, api.PatchGrid((17, 17), (1, 1), 3, True), "swe", 1e-3, 1 / 16, lib=lib)
        assert math.isfinite(api.band_threshold([1, 2], api.ThresholdSpec("capped", 1.0), lib=lib))


def test_metrics_csv_schema(oracle, tmp_path):
    """test_pipeline.cpp:79-95: the metrics file has the documented header and
    one line per row, each formatted as write_metrics_row (pipeline.hpp:78-84)."""
    path = tmp_path / "m.csv"
    cfg = api.RunConfig(scheme="transport", nx=33, splits=(2, 2), levels=3, t_end=0.02,
                        spec=api.ThresholdSpec("capped", 0.01), metrics_path=str(path))
    r = api.run(cfg, lib=oracle)
    lines = path.read_text().splitlines()
    assert lines[0] == "step,time,dense_bytes,compressed_bytes,ratio,nnz,zeroed,global_mass,l2_error"
    assert len([x for x in lines[1:] if x]) == len(r.rows)
    for line, row in zip(lines[1:], r.rows):
        f = line.split(",")
        assert int(f[0]) == row["step"] and float(f[1]) == row["time"] and int(f[5]) == row["nnz"]
        assert float(f[7]) == row["global_mass"] and float(f[8]) == row["l2"]  # %.17g round-trips


@pytest.mark.parametrize("scheme", ["transport", "swe", "lbm"])
def test_lz_metrics_vs_reference(oracle, reference, scheme):
    """Codec::lz (codec.hpp:81-244): the restated greedy parse gives the
    reference's stream sizes byte for byte (compressed_bytes, ratio)."""
    kw = dict(lbm_steps=3) if scheme == "lbm" else dict(t_end=0.005)
    nx = 129 if scheme != "swe" else 65
    cfg = api.RunConfig(scheme=scheme, nx=nx, splits=(2, 2), levels=4 if scheme != "swe" else 3,
                        spec=api.ThresholdSpec("capped", 1e-3), codec="lz", compute_l2=False, **kw)
    a, b = api.run(cfg, lib=oracle), api.run(cfg, lib=reference)
    assert [(r["compressed_bytes"], r["ratio"]) for r in a.rows] == [(r["compressed_bytes"], r["ratio"]) for r in b.rows]


# ---- Codec::lz bytes (codec.hpp:81-244): the C restatement's lz_encode /
# lz_decode against the reference compiled unchanged, byte for byte ----------

def test_lz_codec_matches_reference(oracle, reference):
    from .lz_cases import CHUNKS, corruptions, lz_inputs

    for name, data in lz_inputs().items():
        for chunk in CHUNKS:
            if chunk < 64 and len(data) > 5000:
                continue
            got = api.lz_encode(data, chunk, lib=oracle)
            want = api.lz_encode(data, chunk, lib=reference)
            assert got == want, (name, chunk)
            assert api.lz_decode(got[0], got[1], chunk, len(data), lib=oracle) == data, (name, chunk)
    data = lz_inputs()["smooth_f64"][:4000]
    pl, lens = api.lz_encode(data, 1 << 16, lib=reference)
    for name, p2, l2 in corruptions(pl, lens):
        for lib in (oracle, reference):
            with pytest.raises(abi.CorruptStreamError):
                api.lz_decode(p2, l2, 1 << 16, len(data), lib=lib)
    for lib in (oracle, reference):
        with pytest.raises(abi.InvalidArgument):
            api.lz_encode(b"abc", 0, lib=lib)
