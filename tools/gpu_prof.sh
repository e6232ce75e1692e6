# plain run first (must exit 0), then the launch list and one full capture of k_force
set -x
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_force -s 2 -c 1 -o gpurun_out/force_prof -f $CMD > gpurun_out/ncu_full.log 2>&1
echo rc=$?
