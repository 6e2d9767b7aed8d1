#!/bin/bash
# parity + bench (+ optional ncu of one GEMM shape) in one box call
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/gpu_parity.sh
ENVS="${ENVS:-MTFM_FUSE=0}" bash scripts/gpu_bench_env.sh
if [ -n "$NCU_SHAPE" ]; then
  SHAPE=$NCU_SHAPE MTFM_GEMM_EPI=8 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 5 -c 1 -o gpurun_out/prof_$NCU_SHAPE python scripts/gemm_sweep.py > gpurun_out/ncu_$NCU_SHAPE.log 2>&1
  echo "ncu rc=$?"
fi
