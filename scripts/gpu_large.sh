#!/bin/bash
# large / paper bench lines + one ncu capture of the large-shape residual GEMM (f2_L)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for C in large paper; do
  timeout -s KILL 900 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b_$C.log 2>&1; echo "$C rc=$?"
  grep '^{' gpurun_out/b_$C.log | tail -1 | cut -c1-300
done
SHAPE=f2_L timeout -s KILL 300 python scripts/gemm_sweep.py > gpurun_out/f2L_plain.log 2>&1; tail -2 gpurun_out/f2L_plain.log
SHAPE=f2_L timeout -s KILL 900 ncu -f --set full --clock-control none --import-source on -k regex:gemm_tc -s 3 -c 1 -o gpurun_out/prof_f2L python scripts/gemm_sweep.py > gpurun_out/ncu_f2L.log 2>&1; echo "ncu rc=$?"
