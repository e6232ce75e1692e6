# 1.5M-atom SPC box (BASELINE config 4) at N = 1, 2, 4 (run with gpurun --gpus 4)
A=${ATOMS:-1500000}
timeout 900 python bench.py --atoms $A --steps 20 --warmup 5 --no-cpu-baseline --no-md $EXTRA > gpurun_out/big_n1.json 2> gpurun_out/big_n1.err
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --atoms $A --steps 20 --warmup 5 $EXTRA > gpurun_out/big_n$n.json 2> gpurun_out/big_n$n.err
done
for n in 1 2 4; do python -c "import json; d=json.loads([l for l in open('gpurun_out/big_n$n.json') if l.startswith('{')][0]); print($n, round(d['value']/1e9,2), 'Gpairs/s', round(d['ms_per_step'],4), 'ms/step', 'k_force', round(d['roofline']['kernel_ms']*1e3,1), 'us frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']/1e9,2), 'clocks', d['clocks'])" || tail -5 gpurun_out/big_n$n.err; done
