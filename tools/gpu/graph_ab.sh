#!/bin/bash
cat > /tmp/ab.py <<'PY'
import sys, time, os
sys.path.insert(0, '.')
from paper_2302_09883_b200 import abi, api
lib = abi.load_product()
for name, cfg in [("C1 transport 257^2 100 steps", api.RunConfig(scheme="transport", nx=257, splits=(8, 8), levels=4, t_end=100 / 512, spec=api.ThresholdSpec("capped", 1e-3))),
                  ("LBM 129^2 (4x4 patches of 33) 200 steps", api.RunConfig(scheme="lbm", nx=129, splits=(4, 4), levels=4, lbm_steps=200, spec=api.ThresholdSpec("capped", 1e-3)))]:
    api.run(cfg, lib=lib)
    best = min(api.run(cfg, lib=lib).summary["total_seconds"] for _ in range(5))
    print(("eager " if os.environ.get("WG_NO_GRAPHS") else "graph ") + name, round(best * 1e3, 3), "ms")
PY
python /tmp/ab.py; WG_NO_GRAPHS=1 python /tmp/ab.py
