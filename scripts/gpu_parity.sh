#!/bin/bash
# GPU parity tests, split so a fault in one group does not hide the others.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "fp32 or plan" -p no:cacheprovider > gpurun_out/t_fp32.log 2>&1; echo "fp32 rc=$?"
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "not fp32 and not plan" -p no:cacheprovider > gpurun_out/t_bf16.log 2>&1; echo "bf16 rc=$?"
tail -n 15 gpurun_out/t_fp32.log; tail -n 15 gpurun_out/t_bf16.log
