#!/bin/bash
# SWE change check (run under gpurun): SWE parity tests, then the C3 bench line.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_swe.py tests/test_gpu_bench_configs.py tests/test_gpu_shards.py tests/test_gpu_checkpoint.py \
  tests/test_gpu_session.py -q -x -k "swe or SWE or c3" -p no:cacheprovider --timeout 600 > gpurun_out/quick_swe.log 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/quick_swe.log
timeout 300 python bench.py --workload swe_c3 --no-cpu-baseline > gpurun_out/qb_c3.json 2> gpurun_out/qb_c3.err; echo "c3 rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/qb_c3.json').read().strip().splitlines()[-1]);print('C3', d['value'], d['roofline']['frac'], d['e2e']['value'], d['mass_drift'])"
