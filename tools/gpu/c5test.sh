#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_shards.py -q -k "c5_full" -p no:cacheprovider --timeout 1400 > gpurun_out/c5test.log 2>&1
echo "rc=$?"; tail -30 gpurun_out/c5test.log
