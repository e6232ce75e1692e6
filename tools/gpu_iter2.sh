python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/it_pytest.log 2>&1; tail -2 gpurun_out/it_pytest.log
bash tools/gpu_var.sh
bash tools/gpu_dbg_steps.sh
