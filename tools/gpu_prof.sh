# profiles/ artifacts: plain bench (must exit 0) -> ncu launch list of the same
# command -> one full capture of k_force.  Summarised by tools/summarize_prof.py.
set -x
CMD="python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_force -s 5 -c 1 -o gpurun_out/force_prof -f $CMD > gpurun_out/ncu_full.log 2>&1
echo rc=$?
