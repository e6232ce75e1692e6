# round evidence on one B200 (-> gpurun_out/ev_*): default bench line (moving
# trajectory, CPU baseline, rigid-water MD), static line, reference arm,
# BASELINE configs 1, 2 and 5, the ncu launch list of the default command and
# one full ncu capture of the force kernel (each ncu only after its command ran
# clean without ncu)
set -x
O=gpurun_out
timeout 900 python bench.py > $O/ev_bench.json 2> $O/ev_bench.err; echo rc=$?
timeout 600 python bench.py --positions static --no-md --no-cpu-baseline > $O/ev_static.json 2> $O/ev_static.err; echo rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/ev_ref.json 2> $O/ev_ref.err; echo rc=$?
# config 1: 3k SPC, shifted cutoff Coulomb (reference physics), search + force + 100 MD steps
timeout 600 python bench.py --atoms 3000 --elec cutoff --md-steps 100 --no-cpu-baseline > $O/ev_cfg1.json 2> $O/ev_cfg1.err; echo rc=$?
# config 2: 24k SPC, LJ + reaction field, nstlist 10
timeout 600 python bench.py --atoms 24000 --elec rf --no-cpu-baseline > $O/ev_cfg2.json 2> $O/ev_cfg2.err; echo rc=$?
# config 5: 96k, Verlet-buffer sweep with dynamic pruning (static box so the inner list stays valid; and moving)
for cfg in "10 1.1" "20 1.15" "40 1.2"; do set -- $cfg
  timeout 600 python bench.py --nstlist $1 --rlist $2 --rinner 1.02 --positions static --steps 80 --no-md --no-cpu-baseline > $O/ev_cfg5_static_n$1.json 2> $O/ev_cfg5_static_n$1.err
  timeout 600 python bench.py --nstlist $1 --rlist $2 --steps 80 --md-steps 200 --no-cpu-baseline > $O/ev_cfg5_moving_n$1.json 2> $O/ev_cfg5_moving_n$1.err
done
CMD="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-md"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/ev_launches.csv $CMD > $O/ev_launch.log 2>&1; echo rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_force_h -s 40 -c 1 -o $O/ev_force_prof -f $CMD > $O/ev_ncu_full.log 2>&1; echo rc=$?
echo done
