for n in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2971$n tools/dd_p2p_check.py 96000 > gpurun_out/p2p_n$n.log 2>&1; echo "rc=$?"
  grep "N=" gpurun_out/p2p_n$n.log
done
