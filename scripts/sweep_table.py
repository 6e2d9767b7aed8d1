"""Markdown table of the sweep bench lines (scripts/gpu_sweep.sh)."""
import glob
import json
import os
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
rows = []
for f in sorted(glob.glob(os.path.join(d, "sweep_[0-9]*.json"))):
    try:
        line = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        continue
    c = line.get("config", {})
    rows.append((os.path.basename(f)[:-5], c.get("layers"), c.get("heads"), c.get("kv_heads"), line.get("n_gpus"),
                 line.get("value"), line.get("ms_per_step"), (line.get("e2e") or {}).get("value"),
                 line.get("step_frac_of_bf16_peak"), (line.get("clocks") or {}).get("sm_mhz"),
                 sum(c.get("targets_per_rank", [0]))))
print("| run | layers | H | G | GPUs | targets | targets/s (device) | ms/step | targets/s (e2e) | step frac of bf16 peak | SM MHz |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for r in rows:
    print(f"| {r[0]} | {r[1]} | {r[2]} | {r[3]} | {r[4]} | {r[10]} | {r[5]:.4g} | {r[6]:.3f} | {r[7]:.4g} | {r[8]:.3f} | {r[9]} |")
