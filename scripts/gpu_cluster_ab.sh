#!/bin/bash
# A/B of the CTA-pair B-multicast GEMM schedule (MTFM_GEMM_CLUSTER) on the streaming large shapes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for C in 0 1; do
  MTFM_GEMM_CLUSTER=$C TAG="CLUSTER=$C" timeout -s KILL 300 python scripts/gemm_sweep.py > gpurun_out/clus_$C.log 2>&1; echo "sweep $C rc=$?"
  cat gpurun_out/clus_$C.log | tail -9
done
