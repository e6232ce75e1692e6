CMD="python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
$CMD > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none -k regex:k_search -s 2 -c 1 -o gpurun_out/search_prof -f $CMD > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_prune_entries -s 1 -c 1 -o gpurun_out/prune_prof -f $CMD > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_compact_order -s 1 -c 1 -o gpurun_out/compact_prof -f $CMD > /dev/null 2>&1
echo done
