# DD halo-first force step: 2-GPU tests, exchange-path parity + timing at 2 and 4 GPUs, 1.5M bench lines at 4 GPUs
timeout 600 python -m pytest -q -x tests/test_gpu_dd.py 2>&1 | tail -2
for n in 2 4; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2970$n tools/dd_p2p_check.py 1500000 2>&1 | grep "N="; done
for r in 1 2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2971$r bench.py --gpus 4 --atoms 1500000 --steps 40 --warmup 5 > gpurun_out/hf.json 2> gpurun_out/hf.err
  python -c "import json; d=json.loads([l for l in open('gpurun_out/hf.json') if l.startswith('{')][0]); print('1.5M n4', round(d['value']/1e9,1), 'G', round(d['ms_per_step'],4), 'ms/step')" || tail -3 gpurun_out/hf.err
done
