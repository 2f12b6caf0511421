#!/bin/bash
# GPU test pass (run under gpurun from the repo root) + DSMEM probe.
set -u
mkdir -p gpurun_out
[ -x tools/cuda/dsmem_bulk ] && timeout 60 tools/cuda/dsmem_bulk > gpurun_out/dsmem_bulk.txt 2>&1
cat gpurun_out/dsmem_bulk.txt
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 -p no:cacheprovider > gpurun_out/gputest.log 2>&1
echo "pytest rc=$?"
tail -30 gpurun_out/gputest.log
