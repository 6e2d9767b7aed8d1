#!/bin/bash
cd $GRAFT_REPO_ROOT
for cfg in "MTFM_GEMM_EPI=8" "MTFM_GEMM_EPI=12" ; do
  env $cfg TAG="$cfg" timeout 300 python scripts/gemm_sweep.py 2>&1 | grep -v Warn
done
