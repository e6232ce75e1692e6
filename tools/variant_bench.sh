# bench each library variant in tools/variants/ (kernel time of k_force)
for f in tools/variants/*.so; do
  cp $f paper_1506_00716_b200/libnbx.so
  python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/var.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/var.json')); print('$f', round(d['roofline']['kernel_ms']*1e3,1), 'us frac', round(d['roofline']['frac'],4), 'step', round(d['ms_per_step']*1e3,1))"
done
