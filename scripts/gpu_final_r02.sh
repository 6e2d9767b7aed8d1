#!/bin/bash
# Round-2 closing evidence on one box: gpu test tier, smoke(), reference arm, bench lines
# (small default, base, paper), launch list of one small step, ncu --set full captures.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -rA > gpurun_out/t_gpu_final.log 2>&1; echo "pytest gpu rc=$?"
grep -E "passed|failed" gpurun_out/t_gpu_final.log | tail -n 2
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?"
timeout -s KILL 900 python bench.py --impl reference > gpurun_out/bench_ref_final.json 2> gpurun_out/bench_ref_final.err; echo "ref rc=$?"
timeout -s KILL 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
timeout -s KILL 900 python bench.py --config base --steps 5 --no-cpu-baseline --e2e-steps 5 > gpurun_out/bench_base_final.json 2>&1; echo "base rc=$?"
timeout -s KILL 900 python bench.py --config paper --steps 5 --no-cpu-baseline --e2e-steps 5 > gpurun_out/bench_paper_final.json 2>&1; echo "paper rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/plain_prof.log 2>&1 || { echo "plain failed"; tail gpurun_out/plain_prof.log; exit 1; }
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launches rc=$?"
CMD1="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
for spec in "attn_tc:3:attn" "tok_fused:1:tok" "gemm_tc:10:f2full" "gemm_tc:9:projfull"; do
  IFS=: read -r pat skip tag <<< "$spec"
  timeout -s KILL 900 ncu -f --set full --clock-control none --import-source on -k regex:$pat -s $skip -c 1 -o gpurun_out/prof_r02_$tag $CMD1 > gpurun_out/ncu_r02_$tag.log 2>&1
  echo "$tag rc=$?"
done
