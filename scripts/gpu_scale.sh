#!/bin/bash
# N = 1, 2, 4 bench lines on one box (run with gpurun --gpus 4) + the 2-GPU training test
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/scale_${TAG}_n1.json 2>/dev/null; echo "N=1 rc=$?"
for N in 2 4; do
  timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29520 + N)) bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/scale_${TAG}_n$N.log 2>&1
  echo "N=$N rc=$?"; grep '^{' gpurun_out/scale_${TAG}_n$N.log | tail -1 > gpurun_out/scale_${TAG}_n$N.json
done
timeout -s KILL 600 python -m pytest tests/test_gpu_train.py -q -m gpu -rA -k data_parallel -p no:cacheprovider > gpurun_out/t_train_dp4.log 2>&1; echo "dp test rc=$?"
python - <<'PY'
import json
for n in (1, 2, 4):
    try:
        d = json.load(open(f"gpurun_out/scale_r02_n{n}.json"))
        print(n, round(d["value"] / 1e6, 3), "M targets/s", round(d["ms_per_step"], 3), "ms", d["config"].get("targets_per_rank"), d["clocks"]["sm_mhz"])
    except Exception as e:
        print(n, "failed", e)
PY
