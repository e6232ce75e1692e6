# round evidence: gpu tests, smoke, default bench (+cpu baseline), reference arm, launch list, full k_force_h capture
set -x
python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/rc_pytest.log 2>&1; tail -2 gpurun_out/rc_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rc_smoke.log 2>&1; tail -1 gpurun_out/rc_smoke.log
timeout 900 python bench.py > gpurun_out/rc_bench.json 2> gpurun_out/rc_bench.err; echo rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/rc_ref.json 2> gpurun_out/rc_ref.err; echo rc=$?
CMD="python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/pr_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_force -s 5 -c 1 -o gpurun_out/force_prof -f $CMD > gpurun_out/ncu_full.log 2>&1
echo done
