#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_lz_codec.py tests/test_gpu_lz.py tests/test_gpu_refsuites.py tests/test_gpu_dropin.py -q -p no:cacheprovider --timeout 900 > gpurun_out/lz_tests.log 2>&1
echo "tests rc=$?"; tail -15 gpurun_out/lz_tests.log
