"""Codec::lz (codec.hpp:81-244) in the device session: the store stays CSR
(both codecs are lossless, so the state is the same), and every step's
compressed_bytes / ratio are the byte sizes of lz_encode of the thresholded
coefficient arrays — computed on the device with the reference's greedy
parse and checked EXACTLY against the reference itself (oracle/_ref, the
headers compiled unchanged, run() with Codec::lz)."""
from __future__ import annotations

import pytest

from paper_2302_09883_b200 import api

from .test_gpu_session import compare_runs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize(
    "scheme,nx,splits,levels,mode,c,steps",
    [("transport", 129, (2, 2), 4, "capped", 1e-3, 6),
     ("transport", 129, (4, 4), 3, "constant", 1e-2, 5),
     ("transport", 65, (8, 8), 2, "accumulation", 5e-2, 4),
     ("transport", 129, (2, 2), 4, "capped", 0.0, 3),   # nothing zeroed: skip rule, raw patches
     ("swe", 65, (2, 2), 3, "constant", 5e-4, 8),      # device clock: rows of live steps only
     ("swe", 129, (4, 4), 4, "constant", 1e-3, 5),
     ("lbm", 129, (2, 2), 4, "capped", 1e-3, 4),
     ("lbm", 129, (4, 4), 5, "capped", 1e-5, 3)],
)
def test_lz_metrics_match_reference(product, reference, scheme, nx, splits, levels, mode, c, steps):
    if scheme == "lbm":
        cfg = api.RunConfig(scheme="lbm", nx=nx, splits=splits, levels=levels, lbm_steps=steps,
                            spec=api.ThresholdSpec(mode, c), codec="lz")
    elif scheme == "swe":
        cfg = api.RunConfig(scheme="swe", nx=nx, splits=splits, levels=levels, spec=api.ThresholdSpec(mode, c),
                            codec="lz", t_end=steps * 0.45 / (nx - 1) / 4.5)
    else:
        cfg = api.RunConfig(scheme="transport", nx=nx, splits=splits, levels=levels,
                            spec=api.ThresholdSpec(mode, c), codec="lz", compute_l2=False)
        cfg.t_end = steps * cfg.cfl / (nx - 1) / 0.9
    a, b = api.run(cfg, lib=product), api.run(cfg, lib=reference)
    compare_runs(a, b)  # step, time, bytes (LZ), ratio, nnz, zeroed exact; state bit-exact
    csr = api.run(api.RunConfig(**{**cfg.__dict__, "codec": "csr"}), lib=product)
    assert [r["nnz"] for r in csr.rows] == [r["nnz"] for r in a.rows]
    assert any(r["compressed_bytes"] != s["compressed_bytes"] for r, s in zip(a.rows, csr.rows))
