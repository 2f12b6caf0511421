#!/bin/bash
# One GPU session of measurements (run under gpurun from the repo root):
# bench lines of the default workload and C2/C3, the ncu launch list of the
# default bench command, and the D2Q9 phase profile (tuning build).
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench c4 rc=$?"
tail -c 3000 gpurun_out/bench_c4.json
timeout 300 python bench.py --workload lbm_c2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"
timeout 300 python bench.py --workload swe_c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
if [ -f paper_2302_09883_b200/libwavegrid_b200_prof.so ]; then
  timeout 300 python tools/phase_profile.py --workload lbm_c4 --steps 5 > gpurun_out/phase_c4.txt 2>&1; echo "phase rc=$?"
  cat gpurun_out/phase_c4.txt
fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
