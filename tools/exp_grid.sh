run() { python bench.py --workload $1 --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$2', d['config']['workload'], round(d['value']), 'MLUPS', 'frac', round(d['roofline']['frac'],4), 'launch_ms', round(d['roofline']['avg_launch_ms'],4))"; }
for w in transport_4k_p33 transport_4k; do
  run $w lb2-persist
  WG_GRID_WAVES=100 run $w lb2-full
  WG_PRODUCT_LIB=paper_2302_09883_b200/libwavegrid_b200_lb1.so run $w lb1-persist
  WG_PRODUCT_LIB=paper_2302_09883_b200/libwavegrid_b200_lb1.so WG_GRID_WAVES=100 run $w lb1-full
done
WG_GRID_WAVES=2 run lbm_c2 lbm-waves2
WG_GRID_WAVES=100 run lbm_c2 lbm-full
