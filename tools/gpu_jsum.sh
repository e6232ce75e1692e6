python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/it_pytest.log 2>&1; tail -2 gpurun_out/it_pytest.log
for i in 1 2; do
for v in atomic partials; do
  echo "$v: $(NBX_FORCE_JSUM=$v python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), 'us/step k_force', round(d['roofline']['kernel_ms']*1e3,1), 'e2e', round(d['e2e']['value']/1e9,2))")"
done
done
NBX_BENCH_DEBUG=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 >/dev/null | grep per-step | cut -c1-200
