# one full ncu capture of the force kernel (bench command) for kernel iteration:
#   bash tools/gpu_prof_force.sh [TAG] [ENV=VAL ...]  -> gpurun_out/force_prof_TAG.ncu-rep
TAG=${1:-cur}; shift
CMD="python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
env "$@" $CMD > gpurun_out/pf_plain_$TAG.json 2> gpurun_out/pf_plain_$TAG.err && \
env "$@" ncu --set full --clock-control none --import-source on -k regex:k_force -s 5 -c 1 -o gpurun_out/force_prof_$TAG -f $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo rc=$?
