#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bench_configs.py tests/test_gpu_shards.py -q -k "tiny or l2_sums" -p no:cacheprovider > gpurun_out/newtests.log 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/newtests.log
timeout 300 python tools/phase_profile.py --workload lbm_c4 --steps 5 > gpurun_out/phase_c4.txt 2>&1; cat gpurun_out/phase_c4.txt
