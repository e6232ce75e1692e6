# one full ncu capture of k_force only (bench command), for kernel iteration
CMD="python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
$CMD > gpurun_out/pf_plain.json 2> gpurun_out/pf_plain.err && \
ncu --set full --clock-control none --import-source on -k regex:k_force -s 5 -c 1 -o gpurun_out/force_prof -f $CMD > gpurun_out/ncu_full.log 2>&1
echo rc=$?
