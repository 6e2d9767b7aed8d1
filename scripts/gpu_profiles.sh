#!/bin/bash
# Round-end evidence: bench line, ncu launch list of one bench step, ncu --set full
# of the top kernels (attention, fused tokenizer, one projection GEMM).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo "bench rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/plain_prof.log 2>&1 || { echo "plain failed"; tail gpurun_out/plain_prof.log; exit 1; }
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launches rc=$?"
for spec in "attn_tc:2:attn" "tok_fused:1:tok" "gemm_tc:4:gemm"; do
  IFS=: read -r pat skip tag <<< "$spec"
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:$pat -s $skip -c 1 -o gpurun_out/prof_final_$tag $CMD > gpurun_out/ncu_final_$tag.log 2>&1
  echo "$tag rc=$?"
done
