#!/bin/bash
# ncu --set full of one kernel (regex $1) inside a short bench run; tag $2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/ncu_plain_$2.log 2>&1 || { echo "plain failed"; tail gpurun_out/ncu_plain_$2.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${SKIP:-3} -c 1 -o gpurun_out/prof_$2 $CMD > gpurun_out/ncu_full_$2.log 2>&1
echo "full rc=$?"; tail -2 gpurun_out/ncu_full_$2.log
