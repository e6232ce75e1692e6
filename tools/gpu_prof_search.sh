CMD="python tools/step_breakdown.py --reps 2"
$CMD > gpurun_out/sbp_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_search|k_prune|k_reduce" -s 3 -c 4 -o gpurun_out/search_prof -f $CMD > gpurun_out/sbp_ncu.log 2>&1
echo rc=$?
