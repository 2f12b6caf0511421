#!/bin/bash
# Every bench workload once (run under gpurun): bench lines into gpurun_out/all_<w>.json
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/all_lbm_c4.json 2> gpurun_out/all_lbm_c4.err; echo "lbm_c4 rc=$?"
for w in lbm_c2 swe_c3 lbm_c5 transport_4k transport_4k_p33 transport_c1 lbm_c2_lz lbm_c4_devinit; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/all_$w.json 2> gpurun_out/all_$w.err; echo "$w rc=$?"
done
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/all_reference.json 2> gpurun_out/all_reference.err; echo "ref rc=$?"
for f in gpurun_out/all_*.json; do python - "$f" <<'PY'
import json,sys
f=sys.argv[1]
try:
    d=json.loads(open(f).read().strip().splitlines()[-1])
    r=d.get('roofline') or {}
    print(f.split('all_')[1][:-5], round(d['value'],1), d['unit'], 'frac', round(r.get('frac',0),4), 'e2e', round(d['e2e']['value'],1), 'ratio', round(d.get('compression_ratio',0),2))
except Exception as e:
    print(f, 'ERR', e)
PY
done
