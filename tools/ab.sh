# A/B the default library against variants on the bench workload, interleaved:
#   bash tools/ab.sh "bench args" base VAR ...
# VAR = a tools/variants/VAR/libnbx.so build (tools/build_variant.sh) or
#       KEY=VALUE (an environment setting for the default library)
ARGS=$1; shift
for rep in 1 2; do
  for v in "$@"; do
    LIB=""; ENVS=""
    case "$v" in
      base) ;;
      *=*) ENVS="$v" ;;
      *) LIB=tools/variants/$v/libnbx.so ;;
    esac
    tag=$(echo "$v" | tr '=/' '__')
    env $ENVS NBX_LIB=$LIB timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline $ARGS > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
    python -c "import json,sys; d=json.loads(open('gpurun_out/ab_$tag.json').read().splitlines()[-1]); r=d['roofline']; print('$v', round(d['value']/1e9,1), 'G', round(d['ms_per_step']*1e3,1), 'us/step  k_force', round(r['kernel_ms']*1e3,1), 'us frac', round(r['frac'],3))" || tail -3 gpurun_out/ab_$tag.err
  done
done
