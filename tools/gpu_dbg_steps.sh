for f in tools/variants/*.so; do
  cp $f paper_1506_00716_b200/libnbx.so
  for i in 1 2; do
  NBX_BENCH_DEBUG=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 >/dev/null | grep per-step | cut -c1-300
  done
done
