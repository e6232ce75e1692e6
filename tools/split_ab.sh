timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_edge_cases.py tests/test_gpu_dynamic_prune.py tests/test_gpu_list_step.py 2>&1 | tail -2
NBX_FORCE_SPLIT=4 timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_dynamic_prune.py 2>&1 | tail -2
bash tools/ab.sh "--no-md" base NBX_FORCE_SPLIT=2
bash tools/ab.sh "--no-md --atoms 24000 --elec rf" base NBX_FORCE_SPLIT=1 NBX_FORCE_SPLIT=8
bash tools/ab.sh "--no-md --atoms 3000 --elec cutoff" base NBX_FORCE_SPLIT=1
