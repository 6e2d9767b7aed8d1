#!/bin/bash
# ncu --set full captures only (bench.py must already run on the box)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/plain_prof.log 2>&1 || { echo "plain failed"; tail gpurun_out/plain_prof.log; exit 1; }
for spec in "attn_tc:3:attn" "tok_fused:1:tok" "gemm_tc:10:gemm" "gemm_tc:9:projfull"; do
  IFS=: read -r pat skip tag <<< "$spec"
  timeout -s KILL 900 ncu -f --set full --clock-control none --import-source on -k regex:$pat -s $skip -c 1 -o gpurun_out/prof_final_$tag $CMD > gpurun_out/ncu_final_$tag.log 2>&1
  echo "$tag rc=$?"
done
