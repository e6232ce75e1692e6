# parity tests on the default build, then k_force time per library variant + the legacy kernel
python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/it_pytest.log 2>&1; tail -3 gpurun_out/it_pytest.log
cp paper_1506_00716_b200/libnbx.so /tmp/libnbx_default.so
echo "legacy: $(NBX_FORCE_KERNEL=legacy python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['roofline']['kernel_ms']*1e3,1), 'us frac', round(d['roofline']['frac'],4), 'step', round(d['ms_per_step']*1e3,1))")"
bash tools/variant_bench.sh
cp /tmp/libnbx_default.so paper_1506_00716_b200/libnbx.so
