python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider 2>&1 | tail -2
for i in 1 2; do
echo "pool24: $(python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), 'us k_force', round(d['roofline']['kernel_ms']*1e3,1))")"
echo "pool2: $(NBX_POOL_GB=2 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), 'us k_force', round(d['roofline']['kernel_ms']*1e3,1))")"
done
