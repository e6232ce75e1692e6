# 2 / 4-GPU checks of the migration list step + the bench at 1.5M
timeout 600 python -m pytest -q -x tests/test_gpu_dd.py 2>&1 | tail -2
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 tools/dd_migrate_check.py 96000 2>&1 | grep "PARITY\|Error\|error" | head -5
for n in 2 4; do
  NBX_BENCH_DEBUG=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2958$n bench.py --gpus $n --atoms 1500000 --steps 40 --warmup 5 > gpurun_out/mig_n$n.json 2> gpurun_out/mig_n$n.err
  python -c "import json; d=json.loads([l for l in open('gpurun_out/mig_n$n.json') if l.startswith('{')][0]); print('n$n', round(d['value']/1e9,1), 'G', round(d['ms_per_step'],4), 'ms/step', d['clocks']['sm_mhz'])" || tail -5 gpurun_out/mig_n$n.err
  grep "rank 0 per-step" gpurun_out/mig_n$n.err | cut -c1-200
done
