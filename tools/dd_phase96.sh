for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n tools/dd_breakdown.py 96000 > gpurun_out/ddb96_n$n.log 2>&1
  grep "N=" gpurun_out/ddb96_n$n.log
done
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2956$n tools/dd_breakdown.py 1500000 > gpurun_out/ddb_n$n.log 2>&1
  grep "N=" gpurun_out/ddb_n$n.log | tail -2
done
