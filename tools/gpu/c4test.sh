#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_bench_configs.py -q -k "c4_full" -p no:cacheprovider --timeout 1100 > gpurun_out/c4test.log 2>&1
echo "rc=$?"; tail -30 gpurun_out/c4test.log
