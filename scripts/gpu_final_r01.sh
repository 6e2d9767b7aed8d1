#!/bin/bash
# Round-1 closing evidence on one box: the driver's gpu test tier, smoke(), the
# reference arm, then bench line + launch list + ncu --set full captures.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/t_gpu_all.log 2>&1; echo "pytest gpu rc=$?"
tail -n 5 gpurun_out/t_gpu_all.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout -s KILL 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
bash scripts/gpu_profiles.sh
