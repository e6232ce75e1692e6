# one full ncu capture of the (non-energy) force kernel of the bench command: gpu_prof_k.sh [regex] [out]
K=${1:-k_force}
O=${2:-force_prof}
CMD="python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
$CMD > gpurun_out/pk_plain.json 2> gpurun_out/pk_plain.err || exit 1
ncu --set full --clock-control none --import-source on -k regex:$K -s 5 -c 1 -o gpurun_out/$O -f $CMD > gpurun_out/ncu_$O.log 2>&1
echo rc=$?
