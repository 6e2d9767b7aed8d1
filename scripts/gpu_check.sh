#!/bin/bash
# GPU test tier + smoke + a short bench line on one box.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-chk}
timeout -s KILL 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -rA ${PYTEST_ARGS} > gpurun_out/t_gpu_${TAG}.log 2>&1; echo "pytest gpu rc=$?"
grep -E "passed|failed|error" gpurun_out/t_gpu_${TAG}.log | tail -n 3
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"
timeout -s KILL 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench_${TAG}.json
