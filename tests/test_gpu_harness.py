"""The harness on the device: run() with snapshots and an observer
(test_pipeline.cpp:97-125), transform/restore through the product's per-op
kernels, the demo KAT."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2302_09883_b200 import api, harness

from .test_gpu_session import bits

pytestmark = pytest.mark.gpu


def _small(t_end):
    return api.RunConfig(scheme="transport", nx=33, splits=(2, 2), levels=3, t_end=t_end,
                         spec=api.ThresholdSpec("capped", 0.01))


def test_snapshots_at_requested_times(product, oracle, tmp_path):
    cfg = _small(0.04)
    pre = str(tmp_path / "s_")
    r = harness.run_observed(cfg, [0.0, 0.02, 0.04], pre, lib=product)
    for name in ("s_t0.000.wgrd", "s_t0.020.wgrd", "s_t0.040.wgrd"):
        assert (tmp_path / name).exists()
    comps = harness.load_wgrd(tmp_path / "s_t0.000.wgrd")
    assert len(comps) == 1 and comps[0].shape == (33, 33)
    ic = harness.assemble(api.initial_state(cfg, lib=oracle), 0)  # exact_transport(0)
    assert np.array_equal(bits(comps[0]), bits(ic))
    ref = api.run(cfg, lib=oracle)
    assert [(x["step"], x["time"], x["nnz"]) for x in r.rows] == [(x["step"], x["time"], x["nnz"]) for x in ref.rows]
    assert np.array_equal(bits(r.grid.logical_view()), bits(ref.grid.logical_view()))


@pytest.mark.parametrize("scheme", ["transport", "swe"])
def test_observer_sees_every_step(product, scheme):
    cfg = _small(0.02) if scheme == "transport" else api.RunConfig(
        scheme="swe", nx=33, splits=(2, 2), levels=3, t_end=0.01, spec=api.ThresholdSpec("constant", 5e-4))
    seen = []
    r = harness.run_observed(cfg, observer=lambda g, row: seen.append(row["step"]), lib=product)
    assert seen == list(range(1, len(r.rows) + 1)) and len(seen) > 0


def test_transform_restore_on_device(product, oracle, tmp_path):
    x = np.linspace(0.0, 1.0, 129)
    f = 1.0 + np.exp(-30.0 * ((x[:, None] - 0.5) ** 2 + (x[None, :] - 0.5) ** 2))
    harness.save_wgrd(tmp_path / "in.wgrd", [f, 2.0 * f])
    for lib, tag in ((product, "p"), (oracle, "o")):
        harness.transform_file(tmp_path / "in.wgrd", 5, api.ThresholdSpec("capped", 1e-4), 1, 65536,
                               tmp_path / f"{tag}.wgc", lib=lib)
        harness.restore_file(tmp_path / f"{tag}.wgc", tmp_path / f"{tag}.wgrd", lib=lib)
    assert (tmp_path / "p.wgc").read_bytes() == (tmp_path / "o.wgc").read_bytes()
    assert (tmp_path / "p.wgrd").read_bytes() == (tmp_path / "o.wgrd").read_bytes()


def test_demo_on_device(product):
    rep = harness.demo_discontinuous("", 0.2, lib=product)
    assert rep.nonzeros == 481
