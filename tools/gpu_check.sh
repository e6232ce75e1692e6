set -x
python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu_3.log 2>&1; tail -3 gpurun_out/pytest_gpu_3.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err; echo rc=$?
tail -3 gpurun_out/bench_a.err; cat gpurun_out/bench_a.json
