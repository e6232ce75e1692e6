# rolling-prune check: GPU tests + bench + MD sweep with the rolling prune
python -m pytest tests/test_gpu_dynamic_prune.py tests/test_gpu_engine.py -q --timeout 600 -p no:cacheprovider 2>&1 | tail -4
python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider 2>&1 | tail -2
python bench.py --steps 30 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys;d=json.load(sys.stdin);print(round(d['value']/1e9,1),'G', round(d['ms_per_step']*1e3,1),'us frac',round(d['roofline']['frac'],3),'kern',round(d['roofline']['kernel_ms']*1e3,1))"
for cfg in "10 1.1 0 0" "10 1.1 1.02 2" "20 1.15 0 0" "20 1.15 1.02 2" "40 1.2 0 0" "40 1.2 1.02 2"; do
  set -- $cfg
  python tools/md_bench.py --atoms 288000 --steps 400 --nstlist $1 --rlist $2 --rinner $3 --prune-interval $4 --json 2>&1 | tail -1
done
