python -m pytest tests/test_gpu_dynamic_prune.py -q --timeout 600 -p no:cacheprovider > gpurun_out/dp_pytest.log 2>&1; tail -15 gpurun_out/dp_pytest.log
python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/all_pytest.log 2>&1; tail -3 gpurun_out/all_pytest.log
python bench.py --steps 50 --no-cpu-baseline > gpurun_out/dp_bench.json 2> gpurun_out/dp_bench.err; echo rc=$?
python bench.py --steps 50 --no-cpu-baseline --rinner 0 > gpurun_out/dp_bench0.json 2>> gpurun_out/dp_bench.err; echo rc=$?
python bench.py --steps 80 --no-cpu-baseline --nstlist 40 --rlist 1.2 > gpurun_out/dp_bench40.json 2>> gpurun_out/dp_bench.err; echo rc=$?
tail -3 gpurun_out/dp_bench.err
