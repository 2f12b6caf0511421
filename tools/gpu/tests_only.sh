#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 -p no:cacheprovider > gpurun_out/gputest.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/gputest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/all_lbm_c4.json 2> gpurun_out/all_lbm_c4.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/all_lbm_c4.json').read().strip().splitlines()[-1]);print('C4', d['value'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'])"
