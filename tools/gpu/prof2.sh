#!/bin/bash
# phase profile + one ncu --set full capture of the steady-state C4 step kernel
mkdir -p gpurun_out
timeout 300 python tools/phase_profile.py --workload lbm_c4 --steps 5 > gpurun_out/phase_c4.txt 2>&1; cat gpurun_out/phase_c4.txt
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:k_lbm_pair<.int.65, .int.4, .int.0>" --launch-skip 1 -c 1 -o gpurun_out/r2b_lbm_c4 -f \
  python tools/prof_step.py --workload lbm_c4_devinit --steps 3 > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"; tail -2 gpurun_out/ncu_full.log
