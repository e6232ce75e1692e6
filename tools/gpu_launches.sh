# device time of every kernel launched by tools/step_breakdown.py (ncu launch list)
CMD="python tools/step_breakdown.py --reps 3"
$CMD > gpurun_out/sb_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sb_launches.csv $CMD > gpurun_out/sb_ncu.log 2>&1
echo rc=$?
