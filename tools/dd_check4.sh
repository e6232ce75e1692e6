# 2-GPU DD tests + two 1.5M 4-GPU bench lines + the per-rank force-step trace (gpurun --gpus 4)
timeout 600 python -m pytest -q -x tests/test_gpu_dd.py 2>&1 | tail -2
for rep in 1 2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2956$rep bench.py --gpus 4 --atoms 1500000 --steps 40 --warmup 5 > gpurun_out/ddab.json 2> gpurun_out/ddab.err
  python -c "import json; d=json.loads([l for l in open('gpurun_out/ddab.json') if l.startswith('{')][0]); print('n4', round(d['value']/1e9,1), 'G', round(d['ms_per_step'],4), 'ms/step k_force', round(d['roofline']['kernel_ms']*1e3,1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ddab.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 tools/dd_step_trace.py 1500000 2>&1 | grep -A9 "rank 2:"
