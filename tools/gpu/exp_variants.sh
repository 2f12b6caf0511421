#!/bin/bash
# Timing experiments: bench C4 with tuning-variant libraries (results of
# the experiment variants are NOT valid; timing only).
mkdir -p gpurun_out
for v in "" $WG_VARIANTS; do
  lib=paper_2302_09883_b200/libwavegrid_b200${v:+_$v}.so
  [ -f $lib ] || continue
  WG_PRODUCT_LIB=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/exp_$v.json 2> gpurun_out/exp_$v.err
  python -c "import json;d=json.loads(open('gpurun_out/exp_$v.json').read().strip().splitlines()[-1]);print('variant ${v:-base}', round(d['value'],1), round(d['roofline']['avg_launch_ms'],3))" 2>&1 | tail -1
done
