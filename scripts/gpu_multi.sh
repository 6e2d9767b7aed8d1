#!/bin/bash
# integration test + multi-GPU bench (run with gpurun --gpus N)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout -s KILL 600 python -m pytest tests/test_gpu_integration.py -q -m gpu -p no:cacheprovider > gpurun_out/t_integ.log 2>&1; echo "integ rc=$?"; tail -3 gpurun_out/t_integ.log
if [ "$N" -gt 1 ]; then
  timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/bench_n$N.log 2>&1; echo "bench N=$N rc=$?"
  grep '^{' gpurun_out/bench_n$N.log | tail -1 | cut -c1-400
  timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus $N --steps 2 --warmup 3 > gpurun_out/bench_ref_n$N.log 2>&1; echo "ref N=$N rc=$?"
  grep '^{' gpurun_out/bench_ref_n$N.log | tail -1 | cut -c1-300
fi
