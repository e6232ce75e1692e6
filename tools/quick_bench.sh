# k_force time / frac / step time of the default bench (3 runs)
for i in 1 2 3; do
python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value']/1e9,2), 'G/s  step', round(d['ms_per_step']*1e3,1), 'us  k_force', round(d['roofline']['kernel_ms']*1e3,1), 'us  frac', round(d['roofline']['frac'],4), ' e2e', round(d['e2e']['value']/1e9,2))"
done
