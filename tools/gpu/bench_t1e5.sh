#!/bin/bash
mkdir -p gpurun_out
for w in lbm_c4_t1e5 lbm_c2_t1e5; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --steps 20 > gpurun_out/all_$w.json 2> gpurun_out/all_$w.err; echo "$w rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/all_$w.json').read().strip().splitlines()[-1]);print('$w', round(d['value'],1), round(d['roofline']['frac'],4), round(d['compression_ratio'],2))"
done
timeout 300 python tools/phase_profile.py --workload lbm_c4_t1e5 --steps 5 > gpurun_out/phase_c4_t1e5.txt 2>&1; cat gpurun_out/phase_c4_t1e5.txt
