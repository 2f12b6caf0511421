"""The file/experiment harness (paper_2302_09883_b200/harness.py) against the
reference's own tests: WGRD round trip, transform_file/restore_file
(test_pipeline.cpp:127-158), sweep (160-177), the discontinuous demo
(179-200).  On CPU through the C oracle; the same calls run on the product's
per-op GPU kernels in tests/test_gpu_ops.py-style parity below."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2302_09883_b200 import abi, api, harness


def test_wgrd_round_trip(tmp_path):
    rng = np.random.default_rng(3)
    comps = [rng.standard_normal((17, 33)) for _ in range(3)]
    harness.save_wgrd(tmp_path / "a.wgrd", comps)
    back = harness.load_wgrd(tmp_path / "a.wgrd")
    assert all(np.array_equal(a, b) for a, b in zip(comps, back))
    (tmp_path / "bad.wgrd").write_bytes(b"XGRD" + (tmp_path / "a.wgrd").read_bytes()[4:])
    with pytest.raises(abi.CorruptStreamError):
        harness.load_wgrd(tmp_path / "bad.wgrd")


def test_transform_restore_round_trip(oracle, tmp_path):
    """test_pipeline.cpp:127-158: c = 0 restores the field to round-off; the
    WGC1 bytes equal the reference writer's layout (re-read by load_wgc)."""
    x = np.linspace(0.0, 1.0, 65)
    f = 1.0 + np.exp(-30.0 * ((x[:, None] - 0.5) ** 2 + (x[None, :] - 0.5) ** 2))
    harness.save_wgrd(tmp_path / "in.wgrd", [f])
    harness.transform_file(tmp_path / "in.wgrd", 4, api.ThresholdSpec("constant", 0.0), 1, 65536,
                           tmp_path / "c.wgc", lib=oracle)
    harness.restore_file(tmp_path / "c.wgc", tmp_path / "out.wgrd", lib=oracle)
    back = harness.load_wgrd(tmp_path / "out.wgrd")[0]
    assert np.max(np.abs(back - f)) < 1e-12
    with open(tmp_path / "c.wgc", "rb") as fh:
        p = api.load_wgc(fh)
    assert p.codec == 1 and p.dims == (65, 65) and p.levels == 4 and p.components == 1
    with pytest.raises(ValueError):
        harness.transform_file(tmp_path / "in.wgrd", 4, api.ThresholdSpec("constant", 0.0), 2, 65536,
                               tmp_path / "l.wgc", lib=oracle)


def test_sweep_point_reproduces_run(oracle, tmp_path):
    """test_pipeline.cpp:160-177: a one-point sweep equals the direct run."""
    base = api.RunConfig(scheme="transport", nx=33, splits=(2, 2), levels=3, t_end=0.02,
                         spec=api.ThresholdSpec("capped", 0.01))
    table = harness.sweep(harness.SweepConfig(base, [0.01], [3], [1], str(tmp_path)), lib=oracle)
    direct = api.run(base, lib=oracle)
    assert len(table) == 1 and table[0].avg_ratio == direct.summary["avg_ratio"]
    assert table[0].final_l2 == direct.rows[-1]["l2"]
    lines = (tmp_path / "summary.csv").read_text().splitlines()
    assert lines[0] == "codec,level,threshold,avg_ratio,final_l2_error,metrics_file" and len(lines) == 2
    assert (tmp_path / "run_csr_L3_c0.01.csv").exists()


def test_demo_discontinuous(oracle, tmp_path):
    """test_pipeline.cpp:179-200 / PAPER.md:481: 481 nonzeros; nothing
    thresholded keeps the mass."""
    rep = harness.demo_discontinuous(str(tmp_path), 0.2, lib=oracle)
    assert rep.total == 129 * 129 and rep.nonzeros == 481
    assert rep.coefficient_ratio == pytest.approx(16641 / 481)
    keep = harness.demo_discontinuous("", 0.0, lib=oracle)
    assert keep.mass_after == pytest.approx(keep.mass_before, rel=1e-12)
    assert (tmp_path / "report.txt").exists() and (tmp_path / "original.wgrd").exists()


def test_sweep_with_both_codecs(oracle, tmp_path):
    """sweep over Codec::csr and Codec::lz (pipeline.hpp:360-401): the LZ
    runs report their own (smaller) byte counts, same state."""
    base = api.RunConfig(scheme="transport", nx=33, splits=(2, 2), levels=3, t_end=0.02,
                         spec=api.ThresholdSpec("capped", 0.01))
    table = harness.sweep(harness.SweepConfig(base, [0.01], [3], [1, 2], str(tmp_path)), lib=oracle)
    assert [e.codec for e in table] == [1, 2] and table[0].avg_ratio != table[1].avg_ratio
    assert (tmp_path / "run_lz_L3_c0.01.csv").exists()
