#!/bin/bash
# BASELINE configs[4] sweep: HTA mix x {GQA, MHA} on the multi-scenario workload (1 GPU),
# then the (3:1) GQA point at 2 and 4 GPUs when they are visible.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for mix in 0:1 1:1 3:1 5:1 3:0; do
  for mha in "" "--mha"; do
    tag="sweep_${mix/:/_}${mha:+_mha}"
    timeout -s KILL 600 python bench.py --config sweep --mix $mix $mha --steps 10 --warmup 3 --no-cpu-baseline \
      --e2e-steps 5 > gpurun_out/$tag.json 2> gpurun_out/$tag.err || echo "$tag failed"
  done
done
NG=$(nvidia-smi -L | wc -l)
for n in 2 4; do
  if [ "$NG" -ge "$n" ]; then
    timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 29517 bench.py --gpus $n --config sweep --mix 3:1 --steps 10 --warmup 3 --e2e-steps 5 \
      > gpurun_out/sweep_3_1_n$n.json 2> gpurun_out/sweep_3_1_n$n.err || echo "n$n failed"
  fi
done
python scripts/sweep_table.py gpurun_out
