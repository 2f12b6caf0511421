#!/bin/bash
mkdir -p gpurun_out
for w in lbm_c5 lbm_c2_lz transport_4k transport_c1; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --kernel-name-base demangled -k "regex:k_(lbm_pair|swe_step)<.int.[0-9]+, .int.[0-9]+, .int.[03]>|k_patch_step<.int.[0-9]+, .int.[0-9]+, .int.[0-9]+, .int.0>" --launch-skip 2 -c 1 \
    --csv --log-file gpurun_out/traf_$w.csv python tools/prof_step.py --workload $w --steps 4 > gpurun_out/traf_$w.log 2>&1
  echo "$w rc=$?"
done
