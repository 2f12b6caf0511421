# A/B of WG_SWE_EXACT_CSR at C3; first: python -m paper_2302_09883_b200.build --variant=exact -DWG_SWE_EXACT_CSR=1
run() { python bench.py --workload swe_c3 --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['value']), 'MLUPS', 'ms', round(d['ms_per_step'],4), 'warm', d['warmup'], 'dev_bytes', d.get('device_bytes'))"; }
for i in 1 2 3; do

  WG_PRODUCT_LIB=paper_2302_09883_b200/libwavegrid_b200_exact.so run exact
  run noexact
done
