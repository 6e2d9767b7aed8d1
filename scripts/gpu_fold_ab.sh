#!/bin/bash
# Parity of the folded-GLN1 path, then an A/B over env variants on the bench configs.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
if [ -z "$NO_TESTS" ]; then
timeout -s KILL 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/fold_tests.log 2>&1; echo "tests rc=$?"
tail -n 25 gpurun_out/fold_tests.log
fi
i=0
for CFG in ${CFGS:-small}; do
for V in ${VARIANTS:-MTFM_FOLD=1 MTFM_FOLD=0}; do
  i=$((i+1))
  env ${V//,/ } timeout -s KILL 600 python bench.py --config $CFG --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ab_${i}.log 2>&1
  python - "$CFG" "$V" "$i" <<'PY'
import json, sys
c, v, i = sys.argv[1:4]
line = [l for l in open(f"gpurun_out/ab_{i}.log") if l.startswith("{")]
if not line:
    print(c, v, "failed:", open(f"gpurun_out/ab_{i}.log").read()[-600:]); sys.exit()
d = json.loads(line[-1])
print(c, v, "ms/step %.3f" % d["ms_per_step"], "value %.4e" % d["value"], "e2e %.4e" % d["e2e"]["value"])
print("   ", {k: v for k, v in list(d["stages_ms"].items())[:9]})
PY
done
done
