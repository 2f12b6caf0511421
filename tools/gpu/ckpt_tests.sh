#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_checkpoint.py tests/test_gpu_lz_codec.py tests/test_gpu_harness.py -q -p no:cacheprovider --timeout 900 > gpurun_out/ckpt_tests.log 2>&1
echo "tests rc=$?"; tail -25 gpurun_out/ckpt_tests.log
