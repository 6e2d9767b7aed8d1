#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-gemm}
CMD="python bench.py --steps 1 --warmup 3 --users 512 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/ncu_plain_${TAG}.log 2>&1 || { echo "plain failed"; exit 1; }
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm_tc_kernel<.int.128>" -s 6 -c 4 -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "full rc=$?"; tail -2 gpurun_out/ncu_full_${TAG}.log
