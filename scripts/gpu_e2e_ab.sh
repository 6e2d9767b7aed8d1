#!/bin/bash
# A/B of two prebuilt libraries (abtmp/libA.so, abtmp/libB.so) on the device-timed and e2e ms/step
cd $GRAFT_REPO_ROOT
LIB=paper_2602_11235_b200/libmtfm_cuda.so
cp $LIB abtmp/lib_orig.so
for rep in 1 2 3; do for v in A B; do
  cp abtmp/lib$v.so $LIB
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 30 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4), d['clocks']['sm_mhz'])"
done; done
cp abtmp/lib_orig.so $LIB
