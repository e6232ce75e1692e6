# BASELINE config 5: 96k box, Verlet-buffer sweep nstlist 10/20/40 with
# r_list 1.1/1.15/1.2 and the prune after every rebuild.
#  (1) bench.py (static SPC water, Ewald): what the longer list interval saves
#      in search cost against what the larger buffer adds to the force kernel;
#  (2) tools/md_bench.py (moving LJ fluid: the 96k oxygen sites of a 288k SPC box): how many rebuilds the
#      drift guard (2 d_max > r_list - r_c) forces at each setting.
# Usage (on the GPU box): bash tools/nstlist_sweep.sh  -> gpurun_out/sweep_*.json
mkdir -p gpurun_out
for cfg in "10 1.1" "20 1.15" "40 1.2"; do
  set -- $cfg
  timeout 600 python bench.py --nstlist $1 --rlist $2 --steps 80 --warmup 5 --no-cpu-baseline \
    > gpurun_out/sweep_bench_n$1.json 2> gpurun_out/sweep_bench_n$1.err; echo "bench nstlist=$1 rc=$?"
  timeout 600 python tools/md_bench.py --atoms 288000 --steps 400 --nstlist $1 --rlist $2 --json \
    > gpurun_out/sweep_md_n$1.log 2>&1; echo "md nstlist=$1 rc=$?"
done
