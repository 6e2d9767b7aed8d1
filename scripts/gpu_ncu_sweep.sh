#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SHAPE=${SHAPE:-tok_mlp1} MTFM_GEMM_EPI=8 python scripts/gemm_sweep.py > gpurun_out/sw_plain.log 2>&1 || { echo plain failed; cat gpurun_out/sw_plain.log; exit 1; }
SHAPE=${SHAPE:-tok_mlp1} MTFM_GEMM_EPI=8 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 5 -c 1 -o gpurun_out/prof_sw python scripts/gemm_sweep.py > gpurun_out/ncu_sw.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_sw.log
