# A/B of the 1.5M 4-GPU bench: equal vs count-balanced slabs vs the overlapped force pass (gpurun --gpus 4)
for rep in 1 2; do
for v in "--slabs equal" "--slabs count" "--slabs count OVERLAP"; do
  E=""; A="$v"
  case "$v" in *OVERLAP) E="NBX_DD_OVERLAP=1"; A="--slabs count";; esac
  env $E timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2955$rep bench.py --gpus 4 --atoms 1500000 --steps 40 --warmup 5 $A > gpurun_out/ddab.json 2> gpurun_out/ddab.err
  python -c "import json; d=json.loads([l for l in open('gpurun_out/ddab.json') if l.startswith('{')][0]); print('$v', round(d['value']/1e9,1), 'G', round(d['ms_per_step'],4), 'ms/step k_force', round(d['roofline']['kernel_ms']*1e3,1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ddab.err
done; done
