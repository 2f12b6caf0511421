#!/bin/bash
mkdir -p gpurun_out
w=swe_c3
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --kernel-name-base demangled -k "regex:k_swe_step<.int.65, .int.4, .int.0>" --launch-skip 2 -c 1 \
  --csv --log-file gpurun_out/traf_$w.csv python tools/prof_step.py --workload $w --steps 4 > gpurun_out/traf_$w.log 2>&1
echo "$w rc=$?"
