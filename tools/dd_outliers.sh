# frequency of slow multi-rank runs (96k, 4 GPUs) with and without the NVML clock-sampling thread
for ct in 1 0; do for r in 1 2 3 4 5 6; do
  NBX_BENCH_CLOCK_THREAD=$ct NBX_BENCH_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 298$ct$r bench.py --gpus 4 --atoms 96000 --steps 40 --warmup 5 --no-md > gpurun_out/ol.json 2> gpurun_out/ol.err
  python - <<PY
import json, re
d = json.loads([l for l in open("gpurun_out/ol.json") if l.startswith("{")][0])
t = open("gpurun_out/ol.err").read()
vals = [eval(x) for x in re.findall(r"\[[0-9., ]+\]", t)]
slow = sorted({(i, round(x, 1)) for v in vals for i, x in enumerate(v) if x > 3.0})
print("clock_thread=$ct", round(d["ms_per_step"], 4), "slow steps:", slow)
PY
done; done
