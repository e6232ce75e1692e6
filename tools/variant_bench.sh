# bench each library variant in tools/variants/ (k_force time, step time), twice, interleaved
for rep in 1 2; do
for f in tools/variants/*.so; do
  cp $f paper_1506_00716_b200/libnbx.so
  python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/var.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/var.json')); print('$f', round(d['roofline']['kernel_ms']*1e3,1), 'us frac', round(d['roofline']['frac'],4), 'step', round(d['ms_per_step']*1e3,1), 'clk', d['clocks']['sm_mhz'])"
done
done
