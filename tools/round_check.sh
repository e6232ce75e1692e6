# full GPU check of the current tree: gpu tests, smoke, default bench (with CPU baseline), reference arm
set -x
python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/rc_pytest.log 2>&1; tail -3 gpurun_out/rc_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rc_smoke.log 2>&1; tail -2 gpurun_out/rc_smoke.log
timeout 900 python bench.py > gpurun_out/rc_bench.json 2> gpurun_out/rc_bench.err; echo rc=$?
tail -3 gpurun_out/rc_bench.err; cat gpurun_out/rc_bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/rc_ref.json 2> gpurun_out/rc_ref.err; echo rc=$?
cat gpurun_out/rc_ref.json
