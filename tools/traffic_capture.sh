for w in lbm_c4 transport_c1 transport_4k_p33 lbm_c2_lz lbm_c5; do
  WG_FIXED_WARMUP=3 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_(lbm|patch|swe)_step" --launch-skip 3 -c 1 --csv --log-file gpurun_out/traf_$w.csv \
    python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/traf_$w.log 2>&1
  echo "$w rc=$?"
done
