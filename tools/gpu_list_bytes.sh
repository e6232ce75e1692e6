# per-kernel device time + DRAM bytes of one list step and the force step (bench command, ncu, cold cache)
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/lb_plain.json 2> gpurun_out/lb_plain.err || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:"k_bin|k_scatter|k_colsort|k_bbox|k_search|k_prune_entries|k_compact_order|k_reduce|k_gather|k_force_h|k_local_coords" \
  -c 40 --log-file gpurun_out/list_bytes.csv $CMD > gpurun_out/lb_ncu.log 2>&1
echo rc=$?
