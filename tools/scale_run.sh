# strong scaling of the bench (moving trajectory) at N = 1, 2, 4 on one box, for
# the 96k (config 3) and 1.5M (config 4) SPC boxes (run with gpurun --gpus 4)
# -> gpurun_out/scale_<atoms>_n<N>.json
for A in ${SIZES:-96000 1500000}; do
  timeout 900 python bench.py --atoms $A --steps 40 --warmup 5 --no-cpu-baseline --no-md $EXTRA > gpurun_out/scale_${A}_n1.json 2> gpurun_out/scale_${A}_n1.err
  for n in 2 4; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n --atoms $A --steps 40 --warmup 5 $EXTRA > gpurun_out/scale_${A}_n$n.json 2> gpurun_out/scale_${A}_n$n.err
  done
  for n in 1 2 4; do python -c "import json; d=json.loads([l for l in open('gpurun_out/scale_${A}_n$n.json') if l.startswith('{')][0]); print($A, $n, round(d['value']/1e9,2), 'Gpairs/s', round(d['ms_per_step'],4), 'ms/step', 'k_force', round(d['roofline']['kernel_ms']*1e3,1), 'us frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']/1e9,2), 'clk', d['clocks']['sm_mhz'] if d['clocks'] else None)" || tail -5 gpurun_out/scale_${A}_n$n.err; done
done
