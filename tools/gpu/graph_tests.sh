#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_session.py tests/test_gpu_fuzz.py tests/test_gpu_lz.py tests/test_gpu_bench_configs.py tests/test_gpu_refsuites.py tests/test_gpu_dropin.py -q -p no:cacheprovider --timeout 900 > gpurun_out/graph_tests.log 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/graph_tests.log
python - <<'PY'
import sys, time
sys.path.insert(0, '.')
from paper_2302_09883_b200 import abi, api
lib = abi.load_product()
cfg = api.RunConfig(scheme="transport", nx=257, splits=(8, 8), levels=4, t_end=100 / 512, spec=api.ThresholdSpec("capped", 1e-3))
api.run(cfg, lib=lib)
t0 = time.perf_counter(); r = api.run(cfg, lib=lib); t1 = time.perf_counter()
print("C1 run():", len(r.rows), "steps", round((t1 - t0) * 1e3, 2), "ms wall incl. IC/upload/download;", "device total_seconds", r.summary["total_seconds"])
PY
