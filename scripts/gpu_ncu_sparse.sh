#!/bin/bash
# ncu --set full of the sparse projections of the pruned small model: SKIP=n COUNT=c TAG=name
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --prune ${BENCH_ARGS}"
$CMD > gpurun_out/ncu_plain_${TAG}.log 2>&1 || { echo "plain failed"; tail gpurun_out/ncu_plain_${TAG}.log; exit 1; }
timeout -s KILL 900 ncu -f --set full --clock-control none --import-source on -k regex:gemm_sp -s ${SKIP:-7} -c ${COUNT:-2} \
  -o gpurun_out/ncu_${TAG} $CMD > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_${TAG}.log
