#!/bin/bash
# dense vs 2:4-sparse projections: bench lines of the pruned model (sparse / dense) and the dense model
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in ${CFGS:-small paper}; do
  for mode in "--prune --sparse-mode 2" "--prune --sparse-mode 0"; do
    tag=$(echo "$cfg $mode" | tr ' -' '_')
    timeout -s KILL 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 $mode \
      > gpurun_out/sp_$tag.json 2> gpurun_out/sp_$tag.err
    python - gpurun_out/sp_$tag.json "$cfg $mode" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
st = {k: v for k, v in d["stages_ms"].items() if k.startswith(("proj", "f2", "attn"))}
print(sys.argv[2], round(d["ms_per_step"], 3), d["config"].get("sparse_mma"), d["clocks"]["sm_mhz"], st)
PY
  done
done
