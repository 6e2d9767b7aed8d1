#!/bin/bash
# Paper-shape (d=768, 3 heads of 256, MQA, (3:1)x4) and base-shape evidence:
# bench lines, then ncu --set full of block 0's attention (3 target + 1 full
# layer) and of its full-layer projection / residual GEMMs, plus a launch list.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r02}
for cfg in paper base; do
  timeout -s KILL 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 \
    > gpurun_out/bench_${cfg}_${TAG}.json 2> gpurun_out/bench_${cfg}_${TAG}.err; echo "bench $cfg rc=$?"
done
CMD="python bench.py --config paper --users 64 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/paper_plain_${TAG}.log 2>&1 || { echo "plain failed"; tail gpurun_out/paper_plain_${TAG}.log; exit 1; }
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/paper_launches_${TAG}.csv $CMD > gpurun_out/paper_ncu_launch_${TAG}.log 2>&1; echo "launches rc=$?"
# per profiled process the forward runs 3 (warmup) + 1 (timed) + 1 (profiled) times; capture the first forward
timeout -s KILL 1500 ncu -f --set full --clock-control none --import-source on -k regex:attn_tc -s 0 -c 4 \
  -o gpurun_out/paper_attn_${TAG} $CMD > gpurun_out/paper_ncu_attn_${TAG}.log 2>&1; echo "attn rc=$?"
timeout -s KILL 1500 ncu -f --set full --clock-control none --import-source on -k regex:gemm_tc -s 9 -c 2 \
  -o gpurun_out/paper_gemm_${TAG} $CMD > gpurun_out/paper_ncu_gemm_${TAG}.log 2>&1; echo "gemm rc=$?"
