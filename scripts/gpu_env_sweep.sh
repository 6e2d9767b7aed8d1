#!/bin/bash
# bench stage times under a list of values of one environment switch: VAR=name VALS="a b c" STAGE=regex
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in ${VALS}; do
  env ${VAR}=$v timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 ${BENCH_ARGS} \
    > gpurun_out/sweep_${VAR}_$v.json 2> gpurun_out/sweep_${VAR}_$v.err
  python - "$v" gpurun_out/sweep_${VAR}_$v.json <<'PY'
import json, re, sys, os
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
st = {k: v for k, v in d["stages_ms"].items() if re.search(os.environ.get("STAGE", "."), k)}
print(sys.argv[1], round(d["ms_per_step"], 4), d["clocks"]["sm_mhz"], st)
PY
done
