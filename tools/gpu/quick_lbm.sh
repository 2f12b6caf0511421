#!/bin/bash
# D2Q9 change check (run under gpurun): LBM parity tests, then C4 / C2 bench lines.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_session.py tests/test_gpu_bench_configs.py tests/test_gpu_shards.py \
  tests/test_gpu_lz.py tests/test_gpu_fuzz.py tests/test_gpu_checkpoint.py -q -x -k "lbm or LBM or c2 or c4 or c5 or budget or fuzz or peer or lz" \
  -p no:cacheprovider --timeout 600 > gpurun_out/quick_tests.log 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/quick_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/qb_c4.json 2> gpurun_out/qb_c4.err; echo "c4 rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/qb_c4.json').read().strip().splitlines()[-1]);print('C4', d['value'], d['roofline']['frac'], d['e2e']['value'])"
timeout 300 python bench.py --workload lbm_c2 --no-cpu-baseline > gpurun_out/qb_c2.json 2> gpurun_out/qb_c2.err; echo "c2 rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/qb_c2.json').read().strip().splitlines()[-1]);print('C2', d['value'], d['roofline']['frac'], d['e2e']['value'])"
if [ -f paper_2302_09883_b200/libwavegrid_b200_prof.so ]; then
  timeout 300 python tools/phase_profile.py --workload lbm_c4 --steps 5 > gpurun_out/phase_c4.txt 2>&1; cat gpurun_out/phase_c4.txt
fi
