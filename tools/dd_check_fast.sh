# 2-GPU DD tests, the migration parity check at 4 GPUs, and 96k / 1.5M bench lines at 4 GPUs (gpurun --gpus 4)
timeout 600 python -m pytest -q -x tests/test_gpu_dd.py 2>&1 | tail -2
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29631 tools/dd_migrate_check.py 96000 2>&1 | grep "PARITY"
for A in 96000 1500000; do for r in 1 2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2964$r bench.py --gpus 4 --atoms $A --steps 40 --warmup 5 --no-md > gpurun_out/f4.json 2> gpurun_out/f4.err
  python -c "import json; d=json.loads([l for l in open('gpurun_out/f4.json') if l.startswith('{')][0]); print($A, round(d['value']/1e9,1), 'G', round(d['ms_per_step'],4), 'ms/step')" || tail -3 gpurun_out/f4.err
done; done
