# launch list of the bench command + one full ncu capture of k_force (non-energy step) and k_reduce
CMD="python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
$CMD > gpurun_out/pr_plain.json 2> gpurun_out/pr_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/pr_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_force -s 5 -c 1 -o gpurun_out/force_prof -f $CMD > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_reduce -s 5 -c 1 -o gpurun_out/reduce_prof -f $CMD > gpurun_out/ncu_red.log 2>&1
echo rc=$?
