#!/bin/bash
# bench under several environment settings: ENVS="A=1 B=2;C=3" (';' separates runs)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
IFS=';' read -ra RUNS <<< "${ENVS:-MTFM_FUSE=0}"
i=0
for R in "${RUNS[@]}"; do
  env $R timeout -s KILL 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 ${BENCH_ARGS} > gpurun_out/env_$i.log 2>&1
  python - "$i" "$R" <<'PY'
import json, sys
i, r = sys.argv[1], sys.argv[2]
line = [l for l in open(f"gpurun_out/env_{i}.log") if l.startswith("{")]
if not line:
    print("ENV", r, "failed:", open(f"gpurun_out/env_{i}.log").read()[-600:]); sys.exit()
d = json.loads(line[-1])
print("ENV", r, "ms/step %.3f" % d["ms_per_step"], "value %.3e" % d["value"], "e2e %.3e" % d["e2e"]["value"])
print("   ", d["stages_ms"])
PY
  i=$((i+1))
done
