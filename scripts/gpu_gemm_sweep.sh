#!/bin/bash
# GEMM_CFGS="A=1 B=2;C=3"  SHAPES="proj_full tok_mlp1"
cd $GRAFT_REPO_ROOT
IFS=';' read -ra RUNS <<< "${GEMM_CFGS:-MTFM_GEMM_EPI=8}"
for cfg in "${RUNS[@]}"; do
  for sh in ${SHAPES:-proj_full}; do
    env $cfg SHAPE=$sh TAG="$cfg" timeout 300 python scripts/gemm_sweep.py 2>&1 | grep -v Warn
  done
done
