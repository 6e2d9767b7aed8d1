#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-attn}
CMD="python bench.py --steps 2 --warmup 3 --users 512 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/ncu_plain_${TAG}.log 2>&1 || { echo "plain failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:"attn_tc" -s 3 -c 1 -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "full rc=$?"; tail -2 gpurun_out/ncu_full_${TAG}.log
