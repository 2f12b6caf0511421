#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/c2_sweep.py --steps 1000 --levels 4 5 --out gpurun_out/r2_c2_sweep.json > gpurun_out/sweep.log 2>&1
echo "sweep rc=$?"; tail -20 gpurun_out/sweep.log
