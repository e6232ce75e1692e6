# one full ncu capture of the kernels matching $1 in tools/step_breakdown.py
CMD="python tools/step_breakdown.py --reps 2"
$CMD > gpurun_out/kp_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${2:-0} -c ${3:-2} -o gpurun_out/kprof -f $CMD > gpurun_out/kp_ncu.log 2>&1
echo rc=$?
