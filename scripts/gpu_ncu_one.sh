#!/bin/bash
# ncu --set full (source counters) of one kernel of the small bench: KERNEL=regex SKIP=n TAG=name
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --users ${USERS:-1024} --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/ncu_plain_${TAG}.log 2>&1 || { echo "plain failed"; tail gpurun_out/ncu_plain_${TAG}.log; exit 1; }
timeout -s KILL 900 ncu -f --set full --clock-control none --import-source on -k regex:${KERNEL} -s ${SKIP:-0} -c 1 \
  -o gpurun_out/ncu_${TAG} $CMD > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_${TAG}.log
