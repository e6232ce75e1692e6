# one full ncu capture of each list-step kernel (search passes, prune, compaction) of the bench command
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/pl_plain.json 2> gpurun_out/pl_plain.err || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_search|k_prune_entries|k_compact_order" -s 3 -c 4 -o gpurun_out/list_prof -f $CMD > gpurun_out/ncu_list.log 2>&1
echo rc=$?
