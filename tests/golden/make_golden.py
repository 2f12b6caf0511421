"""Generate the golden fixtures of tests/golden/ from the REFERENCE itself.

Run in the build container, where /root/reference exists:

    make -C oracle ref && python tests/golden/make_golden.py

It loads oracle/_ref/libwg_ref.so (the reference headers compiled unchanged,
oracle/ref_shim.cpp) and records run() outputs and known-answer vectors.
The GPU box has no /root/reference, so tests there compare against these
committed files.  Integers are exact; doubles are stored as their IEEE bit
patterns (hex) so the fixtures pin bits, not decimal renderings.
"""
from __future__ import annotations

import hashlib
import json
import math
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, str(REPO))

from paper_2302_09883_b200 import abi, api  # noqa: E402


def hexd(x: float) -> str:
    return np.float64(x).view(np.uint64).item().to_bytes(8, "big").hex()


def state_hash(grid: api.PatchGrid) -> str:
    return hashlib.sha256(np.ascontiguousarray(grid.logical_view()).tobytes()).hexdigest()


def rows_json(rows):
    out = []
    for r in rows:
        out.append({
            "step": r["step"], "time": hexd(r["time"]), "dense_bytes": r["dense_bytes"],
            "compressed_bytes": r["compressed_bytes"], "ratio": hexd(r["ratio"]), "nnz": r["nnz"],
            "zeroed": r["zeroed"], "global_mass": hexd(r["global_mass"]), "l2": hexd(r["l2"]),
        })
    return out


def run_golden(ref, name, cfg: api.RunConfig, extra=None):
    res = api.run(cfg, lib=ref)
    last = res.rows[-1]
    doc = {
        "generated_by": "oracle/_ref/libwg_ref.so (reference headers, -O3, no -march)",
        "config": {k: (v.__dict__ if hasattr(v, "__dict__") else v) for k, v in cfg.__dict__.items()},
        "steps": len(res.rows),
        "avg_ratio": res.summary["avg_ratio"],
        "avg_ratio_hex": hexd(res.summary["avg_ratio"]),
        "final": {"nnz": last["nnz"], "zeroed": last["zeroed"], "compressed_bytes": last["compressed_bytes"],
                  "global_mass": last["global_mass"], "l2": last["l2"]},
        "rows": rows_json(res.rows),
        "state_sha256": state_hash(res.grid),
    }
    if extra:
        doc.update(extra)
    (HERE / f"{name}.json").write_text(json.dumps(doc, indent=1) + "\n")
    print(name, len(res.rows), "steps, final", doc["final"])


def demo_field(n=129):
    """pipeline.hpp:421-431 sampled with the C library's exp/sin (math.*)."""
    f = np.empty((n, n))
    for i in range(n):
        for j in range(n):
            x, y = i / n, j / n
            stp = 1.0 if (y - x * x) >= 0.0 else 2.0
            f[i, j] = math.exp(x - y) * math.sin(2.0 * math.pi * (x + y)) * stp
    return f


def main():
    ref = abi.Lib(REPO / "oracle" / "_ref" / "libwg_ref.so")
    assert ref.name == "reference"

    # C1: 256^2 cells, 8x8 patches, L4, capped 1e-3, 100 steps
    run_golden(ref, "c1_transport", api.RunConfig(scheme="transport", nx=257, splits=(8, 8), levels=4,
                                                  t_end=100 / 512, spec=api.ThresholdSpec("capped", 1e-3)))
    # test_pipeline.cpp small_transport()
    run_golden(ref, "small_transport", api.RunConfig(scheme="transport", nx=33, splits=(2, 2), levels=3,
                                                     t_end=0.05, spec=api.ThresholdSpec("capped", 0.01)))
    # test_pipeline.cpp:202-217 dam break
    run_golden(ref, "small_swe", api.RunConfig(scheme="swe", nx=33, splits=(2, 2), levels=3, t_end=0.05,
                                               spec=api.ThresholdSpec("constant", 0.0005)))
    # builder D2Q9 on the reference's compression machinery (parity unpinned by the reference itself)
    run_golden(ref, "small_lbm", api.RunConfig(scheme="lbm", nx=129, splits=(4, 4), levels=4, lbm_steps=20,
                                               spec=api.ThresholdSpec("capped", 1e-3)))

    # known-answer vectors for the transform / threshold / codec
    f = demo_field()
    cs = api.dwt_nd(f, 6, lib=ref)
    z = api.apply_threshold(cs, 6, api.ThresholdSpec("constant", 0.2), lib=ref)
    nnz = int(np.count_nonzero(cs))
    rec = api.idwt_nd(cs, 6, lib=ref)
    blk = api.csr_encode(cs, 129, 129, lib=ref)
    kat = {
        "demo": {
            "n": 129, "levels": 6, "threshold": 0.2, "nonzeros": nnz, "zeroed": z,
            "field_sha256": hashlib.sha256(f.tobytes()).hexdigest(),
            "coeff_sha256": hashlib.sha256(cs.tobytes()).hexdigest(),  # after thresholding
            "recon_sha256": hashlib.sha256(rec.tobytes()).hexdigest(),
            "csr_v_sha256": hashlib.sha256(blk.v.tobytes()).hexdigest(),
            "csr_col_sha256": hashlib.sha256(blk.col.tobytes()).hexdigest(),
            "csr_row_sha256": hashlib.sha256(blk.row.tobytes()).hexdigest(),
        },
    }
    rng = np.random.default_rng(2302)
    x = rng.uniform(-1, 1, (33, 33))
    c33 = api.dwt_nd(x, 4, lib=ref)
    kat["random33_L4"] = {
        "seed": 2302, "input_sha256": hashlib.sha256(x.tobytes()).hexdigest(),
        "coeff_sha256": hashlib.sha256(c33.tobytes()).hexdigest(),
        "recon_sha256": hashlib.sha256(api.idwt_nd(c33, 4, lib=ref).tobytes()).hexdigest(),
    }
    t = c33.copy()
    kat["random33_L4"]["capped_0.05_zeroed"] = api.apply_threshold(t, 4, api.ThresholdSpec("capped", 0.05), lib=ref)
    kat["random33_L4"]["capped_0.05_sha256"] = hashlib.sha256(t.tobytes()).hexdigest()
    (HERE / "kat.json").write_text(json.dumps(kat, indent=1) + "\n")
    print("demo nonzeros", nnz)


if __name__ == "__main__":
    main()
