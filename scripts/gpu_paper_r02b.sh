#!/bin/bash
# Paper-shape evidence after the split K/V rings: bench line, ncu --set full of block 0's
# full-layer and one target-layer attention launch, base and large bench lines.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r02b}
timeout -s KILL 900 python bench.py --config paper --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 \
  > gpurun_out/bench_paper_${TAG}.json 2> gpurun_out/bench_paper_${TAG}.err; echo "bench paper rc=$?"
CMD="python bench.py --config paper --users 64 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/paper_plain_${TAG}.log 2>&1 || { echo "plain failed"; tail gpurun_out/paper_plain_${TAG}.log; exit 1; }
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/paper_launches_${TAG}.csv $CMD > gpurun_out/paper_ncu_launch_${TAG}.log 2>&1; echo "launches rc=$?"
timeout -s KILL 900 ncu -f --set full --clock-control none --import-source on -k regex:attn_tc -s 0 -c 4 \
  -o gpurun_out/paper_attn_${TAG} $CMD > gpurun_out/paper_ncu_attn_${TAG}.log 2>&1; echo "attn rc=$?"
for cfg in base large; do
  timeout -s KILL 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 \
    > gpurun_out/bench_${cfg}_${TAG}.json 2> gpurun_out/bench_${cfg}_${TAG}.err; echo "bench $cfg rc=$?"
done
