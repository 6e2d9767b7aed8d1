#!/bin/bash
# A/B of the fused-producer switches (MTFM_FUSE) on the small workload.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for F in ${FUSES:-0 1 2 3}; do
  MTFM_FUSE=$F timeout -s KILL 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ab_$F.log 2>&1
  python - "$F" <<'PY'
import json, sys
f = sys.argv[1]
line = [l for l in open(f"gpurun_out/ab_{f}.log") if l.startswith("{")]
if not line:
    print("FUSE", f, "failed:", open(f"gpurun_out/ab_{f}.log").read()[-400:]); sys.exit()
d = json.loads(line[-1])
print("FUSE", f, "ms/step %.3f" % d["ms_per_step"], "value %.3e" % d["value"], "e2e %.3e" % d["e2e"]["value"])
print("   ", d["stages_ms"])
PY
done
