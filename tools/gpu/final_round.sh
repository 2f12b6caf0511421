#!/bin/bash
# The whole GPU test suite, every bench workload, the ncu launch list of the
# default bench command and one --set full capture of the C4 step kernel.
set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 -p no:cacheprovider > gpurun_out/gputest.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/gputest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
bash tools/gpu/bench_all.sh
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:k_lbm_pair<.int.65, .int.4, .int.0>" --launch-skip 1 -c 1 -o gpurun_out/r2f_lbm_c4 -f \
  python tools/prof_step.py --workload lbm_c4_devinit --steps 3 > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
