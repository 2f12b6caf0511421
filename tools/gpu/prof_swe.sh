#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:k_swe_step<.int.65, .int.4, .int.0>" --launch-skip 2 -c 1 -o gpurun_out/r2_swe_c3 -f \
  python tools/prof_step.py --workload swe_c3 --steps 4 > gpurun_out/ncu_swe.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_swe.log
