#!/bin/bash
# multi-GPU bench lines at N=2 and N=4 on one 4-GPU box (run with gpurun --gpus 4)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for N in 2 4; do
  timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29510+N)) bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/bench_n$N.log 2>&1; echo "bench N=$N rc=$?"
  grep '^{' gpurun_out/bench_n$N.log | tail -1 | cut -c1-300
  timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29520+N)) bench.py --impl reference --gpus $N --steps 2 --warmup 3 > gpurun_out/bench_ref_n$N.log 2>&1; echo "ref N=$N rc=$?"
  grep '^{' gpurun_out/bench_ref_n$N.log | tail -1 | cut -c1-300
done
