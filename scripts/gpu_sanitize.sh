#!/bin/bash
# compute-sanitizer racecheck + synccheck (+ memcheck) over the bf16 tensor-core
# pipelines (tokenizer, GEMM, attention: mbarrier / TMEM hand-offs) on tiny_j and small4_j.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for fx in tiny_j small4_j; do
  for tool in racecheck synccheck memcheck; do
    timeout -s KILL 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_run.py $fx bf16 \
      > gpurun_out/san_${tool}_${fx}.log 2>&1
    echo "$tool $fx rc=$?"; tail -n 3 gpurun_out/san_${tool}_${fx}.log
  done
done
