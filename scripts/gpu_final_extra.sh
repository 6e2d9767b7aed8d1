#!/bin/bash
# closing evidence part 2: sparse vs dense lines and the large-config line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CFGS="small paper" bash scripts/gpu_sparse_bench.sh
timeout -s KILL 1200 python bench.py --config large --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/bench_large_final.json 2> gpurun_out/bench_large_final.err; echo "large rc=$?"
