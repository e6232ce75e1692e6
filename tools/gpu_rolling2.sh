# MD (96k LJ sites) with dynamic pruning: r_inner / rolling-prune interval sweep
for cfg in "10 1.1 0 0" "10 1.1 1.05 0" "10 1.1 1.05 3" "20 1.15 1.05 3" "40 1.2 0 0" "40 1.2 1.05 3" "40 1.2 1.08 5" "40 1.2 1.05 0"; do
  set -- $cfg
  python tools/md_bench.py --atoms 288000 --steps 400 --nstlist $1 --rlist $2 --rinner $3 --prune-interval $4 --json 2>&1 | tail -1
done
