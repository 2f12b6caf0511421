#!/bin/bash
# D2Q9 phase profile of the tuning build (WG_PHASE_TIMING) at C4 and C2.
mkdir -p gpurun_out
timeout 300 python tools/phase_profile.py --workload lbm_c4 --steps 5 > gpurun_out/phase_c4.txt 2>&1; cat gpurun_out/phase_c4.txt
timeout 300 python tools/phase_profile.py --workload lbm_c2 --steps 20 > gpurun_out/phase_c2.txt 2>&1; cat gpurun_out/phase_c2.txt
