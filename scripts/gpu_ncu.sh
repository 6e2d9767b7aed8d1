#!/bin/bash
# ncu evidence: per-launch device times (launch list) + one --set full capture
# of the top kernels. The same command first runs plain and must exit 0.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r01}
CMD="python bench.py --steps 2 --warmup 3 --users 256 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/ncu_plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"gemm_tc|attn_tc|gln_kernel|gate_kernel|heads_kernel|plan_kernel" -s 20 -c 12 -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "full rc=$?"
tail -3 gpurun_out/ncu_full_${TAG}.log
