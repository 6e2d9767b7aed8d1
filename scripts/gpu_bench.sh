#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 --profile-json gpurun_out/prof.json > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -n 5 gpurun_out/bench.log
