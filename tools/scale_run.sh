# bench at N = 1, 2, 4 on one box (run with gpurun --gpus 4)
python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/scale_n1.json 2>/dev/null
for n in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n --steps 40 --warmup 5 $EXTRA > gpurun_out/scale_n$n.json 2> gpurun_out/scale_n$n.err
done
for n in 1 2 4; do python -c "import json; d=json.loads([l for l in open('gpurun_out/scale_n$n.json') if l.startswith('{')][0]); print($n, round(d['value']/1e9,2), 'Gpairs/s', round(d['ms_per_step'],4), 'ms/step', 'k_force', round(d['roofline']['kernel_ms']*1e3,1), 'us e2e', round(d['e2e']['value']/1e9,2))"; done
