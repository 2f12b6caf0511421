#!/bin/bash
# ncu captures (run under gpurun from the repo root, one GPU): DSMEM duplex
# probe, one `--set full` capture of the steady-state D2Q9 step kernel at C4,
# per-launch DRAM traffic of the step kernels, and the drop-in suites.
set -u
mkdir -p gpurun_out
timeout 120 python tools/prof_step.py --workload lbm_c4_devinit --steps 3 > gpurun_out/prof_plain.log 2>&1
echo "plain rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:k_lbm_pair<.int.65, .int.4, .int.0>" --launch-skip 1 -c 1 -o gpurun_out/r2_lbm_c4 -f \
  python tools/prof_step.py --workload lbm_c4_devinit --steps 3 > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"; tail -3 gpurun_out/ncu_full.log
for w in lbm_c4_devinit lbm_c2 swe_c3 transport_4k_p33; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --kernel-name-base demangled -k "regex:k_(lbm_pair|swe_step)<.int.[0-9]+, .int.[0-9]+, .int.0>|k_patch_step<.int.[0-9]+, .int.[0-9]+, .int.[0-9]+, .int.0>" --launch-skip 2 -c 1 \
    --csv --log-file gpurun_out/traf_$w.csv python tools/prof_step.py --workload $w --steps 4 > gpurun_out/traf_$w.log 2>&1
  echo "$w rc=$?"
done
