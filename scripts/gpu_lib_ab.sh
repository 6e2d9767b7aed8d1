#!/bin/bash
# A/B of prebuilt library variants on one box: abtmp/lib<V>.so copied into place in turn
# (VARIANTS="A B", CFGS="small base", REPS=2, STAGES regex); stage times of each bench line.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
LIB=paper_2602_11235_b200/libmtfm_cuda.so
cp $LIB abtmp/lib_orig.so
for cfg in ${CFGS:-small}; do
  for rep in $(seq ${REPS:-2}); do
    for v in ${VARIANTS:-A B}; do
      cp abtmp/lib$v.so $LIB
      timeout -s KILL 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ab_${cfg}_$v.json 2>/dev/null
      python - $cfg $v gpurun_out/ab_${cfg}_$v.json <<'PY'
import json, os, re, sys
d = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
st = {k: v for k, v in d["stages_ms"].items() if re.search(os.environ.get("STAGES", "attn"), k)}
print(sys.argv[1], sys.argv[2], round(d["ms_per_step"], 4), d["clocks"]["sm_mhz"], st)
PY
    done
  done
done
cp abtmp/lib_orig.so $LIB
