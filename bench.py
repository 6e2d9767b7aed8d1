"""bench.py — scored targets/sec of the MTFM forward (BASELINE.json metric).

Workload (BASELINE.json configs[1], "MTFM-small"): d=256, 8 Q / 2 KV heads,
(3:1)x1 HTA stack (4 layers), 1024 users per GPU x (2 x 224 historical + 64
realtime) context tokens + 4 scenarios x 8 targets, synthetic data, random
weights, bf16 tensor cores. One step = one forward over the whole batch:
planning -> tokenizer -> 4 HTA layers -> MMoE heads -> records.

value : targets/s over all ranks, batch resident in HBM, CUDA events on the
        library stream around exactly K steps, max over ranks (weak scaling:
        every rank scores its own 1024 users; no collective on the data path).
e2e   : the same metric through mtfm_cuda_forward with pinned host buffers:
        H2D of the packed batch, the forward, D2H of the records, every step.
roofline: the dominant stage of a profiled step (CUDA events around each
        stage, same stream), algorithmic FLOPs / its duration
        vs MEASURED_PEAKS.json.
cpu_baseline: the reference CPU path (ref_bench over the unmodified reference
        sources, built on this host with the reference's -march=native when g++
        and baseline/_ref/proj are present, else the x86-64-v3 oracle/_ref build)
        on this host's cores, on the first --ref-users users of the GPU arm's own
        batch (MTFMPB1 file: byte-identical inputs) with the GPU arm's weights.

--impl reference runs only the reference CPU path (rank 0; other ranks exit).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
REF_BENCH = os.path.join(ROOT, "oracle", "_ref", "ref_bench")
REF_SRC = os.path.join(ROOT, "baseline", "_ref", "proj")

# BASELINE.json configs (paper_2602_11235_b200/datagen.py WORKLOADS): small is
# configs[1] (the 1-GPU headline), base configs[2] (heavy-tailed lengths),
# large configs[3] (per-GPU shard), paper the north_star's paper-scale shape.
CONFIGS = ("small", "base", "large", "paper", "sweep")


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_tag():
    """Model name + ISA flags: a -march=native binary is only reused on an identical CPU."""
    import hashlib
    flags = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    flags = line
                    break
    except OSError:
        pass
    return hashlib.sha1((cpu_model() + flags).encode()).hexdigest()[:12]


def ref_bench_binary():
    """(path, how): the reference CPU path built on this host with the reference's own
    -march=native (proj/src/CMakeLists.txt:10-13), cached per CPU model; else the
    x86-64-v3 build that travelled with the snapshot."""
    import shutil
    tag = cpu_tag()
    native = os.path.join(ROOT, "baseline", "_ref", "bin", f"ref_bench_native_{tag}")
    if os.path.exists(native):
        return native, "-march=native (built on this host)"
    why = None
    if not os.path.isdir(REF_SRC):
        why = "baseline/_ref/proj missing"
    elif shutil.which("g++") is None:
        why = "no g++ on this host"
    else:
        os.makedirs(os.path.dirname(native), exist_ok=True)
        r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "native", "REF=" + REF_SRC,
                            "OUT=" + os.path.dirname(native)], capture_output=True, text=True, timeout=600)
        built = os.path.join(os.path.dirname(native), "ref_bench_native")
        if r.returncode == 0 and os.path.exists(built):
            os.replace(built, native)
            return native, "-march=native (built on this host)"
        why = "native build failed: " + r.stderr.strip()[-200:]
    return REF_BENCH, f"-march=x86-64-v3 (prebuilt; {why})"


def write_cpu_inputs(batch, schemas, cfg, params, order):
    """The GPU arm's batch and weights as MTFMPB1 / MTFMPF1 files for ref_bench."""
    import tempfile
    from paper_2602_11235_b200 import packed_io
    d = tempfile.mkdtemp(prefix="mtfm_ref_")
    bp, pp = os.path.join(d, "batch.bin"), os.path.join(d, "params.bin")
    packed_io.save_packed(bp, batch, schemas, cfg)
    packed_io.save_params(pp, params, order)
    return bp, pp


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), d.get("bf16_tflops_sustained", 1400.0), \
            "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and "Active" in r[3 + i]
                          and "Not" not in r[3 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_baseline(inputs, threads, users, reps=2):
    exe, how = ref_bench_binary()
    if not os.path.exists(exe):
        return None
    bp, pp = inputs
    cmd = [exe, "--batch", bp, "--params", pp, "--users", str(users), "--threads", str(threads), "--reps", str(reps)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    if out.returncode != 0:
        return {"error": out.stderr.strip()[-200:]}
    lines = [json.loads(x) for x in out.stdout.strip().splitlines() if x.startswith("{")]
    best = max(lines, key=lambda r: r["targets_per_sec"])
    best["per_rep"] = [r["targets_per_sec"] for r in lines]
    best["build"] = how
    return best


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload_inputs(args):
    """The N=1 batch of the config (the GPU arm's rank-0 input at N=1) and its weights."""
    from paper_2602_11235_b200 import datagen
    from paper_2602_11235_b200.schema import param_specs
    wl = datagen.with_mix(datagen.WORKLOADS[args.config](), args.mix, args.mha)
    batch = datagen.generate(wl, n_users=args.users or wl.n_users)
    specs = param_specs(wl.schemas, wl.cfg)
    params = datagen.random_params(specs, seed=7)
    if getattr(args, "prune", False):
        # the reference arm's copy of the pruned weights: prune_model_projections restated
        # (oracle/mtfm_oracle.py, bit-exact with the reference and the device prune)
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import mtfm_oracle as O
        params = {k: (O.prune_2_4(v)[0] if O.is_projection_param(k) else v) for k, v in params.items()}
    return wl, batch, params, [n for n, _, _ in specs]


def run_reference(args, world, rank):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    users = args.ref_users
    t0 = time.time()
    wl, batch, params, order = workload_inputs(args)
    inputs = write_cpu_inputs(batch, wl.schemas, wl.cfg, params, order)
    rows = []
    for _ in range(args.warmup + args.steps):
        r = cpu_baseline(inputs, threads, users, reps=1)
        if r is None or "error" in (r or {}):
            print(json.dumps({"impl": "reference", "unavailable": f"oracle/_ref/ref_bench missing or failed: {r}"}))
            return
        rows.append(r)
    timed = rows[args.warmup:]
    secs = sum(r["seconds"] for r in timed)
    targets = sum(r["targets"] for r in timed)
    value = targets / secs
    line = {
        "impl": "reference", "metric": "scored targets/sec (device-timed)", "value": value, "unit": "targets/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * secs / len(timed),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"MTFM-{args.config}", "users_per_step": users, "threads": threads,
                   **({"pruned_2_4": True} if args.prune else {}),
                   "cpu_model": cpu_model(), "build": rows[-1].get("build"),
                   "note": "reference Model<float>::forward_sample striped over std::thread workers "
                           "(train.hpp:157-170), compiled from the unmodified reference sources; inputs are "
                           "the first users of the GPU arm's N=1 batch (same bytes) with its weights"},
        "cpu_baseline": {"value": value, "unit": "targets/s", "cores": threads, "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": f"first {users} users of the MTFM-{args.config} batch x {args.steps} steps"},
        "e2e": {"value": value, "unit": "targets/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.time() - t0,
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="small", choices=CONFIGS)
    ap.add_argument("--users", type=int, default=None, help="users per GPU (default: the config's)")
    ap.add_argument("--e2e-steps", type=int, default=50, help="e2e steps per API (pipelined and synchronous)")
    ap.add_argument("--ref-users", type=int, default=96)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-json", default=None)
    ap.add_argument("--mix", default=None, help='HTA mix "K:P" (target:full layers per block), default the config\'s')
    ap.add_argument("--mha", action="store_true", help="kv_heads = heads (no GQA), the reference bench's G=H arm")
    ap.add_argument("--prune", action="store_true",
                    help="2:4-prune f1/fuq/fkv/f2 (prune_projections) before timing: the pruned model")
    ap.add_argument("--sparse-mode", type=int, default=2, choices=[0, 1, 2],
                    help="with --prune: 2:4 sparse tensor cores 2 auto / 1 required / 0 dense (mtfm_cuda_set_sparse_mma)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = dist_setup()
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2602_11235_b200 import Model, abi, datagen
    from paper_2602_11235_b200.schema import BATCH_KEYS, batch_nbytes

    wl = datagen.with_mix(datagen.WORKLOADS[args.config](), args.mix, args.mha)
    per_gpu = args.users or wl.n_users
    if world == 1:
        batch = datagen.generate(wl, n_users=per_gpu)
    else:
        # one global batch of world x per_gpu users, sharded by LPT on each user's
        # algorithmic cost under this model config; no collective touches the data
        # path (weak scaling)
        from paper_2602_11235_b200.shard import shard_plan, take_users
        full = datagen.generate(wl, n_users=per_gpu * world)
        batch = take_users(full, shard_plan(full, world, cfg=wl.cfg)[rank])
        del full
    model = Model(wl.schemas, wl.cfg, precision="bf16", device=local)
    params = datagen.random_params(model.param_specs(), seed=7)
    model.set_params(params)
    sparse_active = None
    if args.prune:
        model.prune_projections()
        sparse_active = model.set_sparse_mma(args.sparse_mode)
        params = {n: model.get_param(n, r, c) for n, r, c in model.param_specs()}  # the CPU arm's weights
    n_targets = int(len(batch["exp_ts"]))
    n_tokens = int(len(batch["ev_ts"])) + n_targets
    rank_targets = [n_targets]
    if dist is not None:
        t = torch.tensor([n_targets], device="cuda", dtype=torch.int64)
        g = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(g, t)
        rank_targets = [int(x.item()) for x in g]
    total_targets = sum(rank_targets)

    stream = torch.cuda.ExternalStream(model.stream_handle(), device=torch.device("cuda", local))

    def barrier():
        if dist is not None:
            dist.barrier()

    # ---------------- device-timed headline (batch resident in HBM)
    pb = model.prepare(batch)
    for _ in range(args.warmup):
        pb.run()
    res = pb.results()
    stats = model.last_stats()
    launches_per_step = int(stats.kernel_launches)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            pb.run()
        ev1.record(stream)
        ev1.synchronize()
        # keep the sampler alive over a short tail so a fast region still gets samples
        t_end = time.time() + 0.3
        while time.time() < t_end and len(clk.rows) < 3:
            pb.run()
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    barrier()
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = total_targets / (ms / 1000.0)  # every rank's targets over the slowest rank's time

    # ---------------- profiled step: per-stage device times (roofline)
    model.set_profiling(True)
    pb.run()
    pb.results()
    prof = model.profile()
    model.set_profiling(False)
    stages = {}
    for name, sms, fl, by in prof:
        s = stages.setdefault(name, [0.0, 0.0, 0.0, 0])
        s[0] += sms
        s[1] += fl
        s[2] += by
        s[3] += 1
    total_prof = sum(v[0] for v in stages.values())
    top = max(stages.items(), key=lambda kv: kv[1][0])
    hbm, tflops, tflops_sus, peak_kind = load_peaks()
    tname, (tms, tfl, tby, tcnt) = top
    if tfl > 0:
        achieved = tfl / (tms / 1000.0) / 1e12
        roof = {"bound": "tensor", "kernel": tname, "achieved": achieved, "peak": tflops, "unit": "TFLOP/s",
                "frac": achieved / tflops, "traffic": None, "launches": tcnt,
                "per_launch_ms": tms / tcnt, "algorithmic_per_launch": tfl / tcnt,
                "share_of_step": tms / total_prof, "peak_kind": peak_kind}
    else:
        achieved = tby / (tms / 1000.0) / 1e9
        roof = {"bound": "hbm", "kernel": tname, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": None, "launches": tcnt, "per_launch_ms": tms / tcnt,
                "algorithmic_per_launch": tby / tcnt, "share_of_step": tms / total_prof, "peak_kind": peak_kind}
    if tname.startswith("attn") and tfl > 0:
        # attention weights are silu(QK^T): one MUFU.TANH per visible (head, query, key) score,
        # 4 * d_h flops each, against the SFU's 16 ops/clk/SM (scripts/ubench_silu.cu)
        dh = wl.cfg.hta.d_model // wl.cfg.hta.heads
        sfu_ops = tfl / (4.0 * dh)
        sfu_peak = 16.0 * 148 * 1.965e9
        sfu_ach = sfu_ops / (tms / 1000.0)
        ceiling = sfu_peak * 4.0 * dh / (tflops * 1e12)
        roof["sfu"] = {"achieved_Gops": sfu_ach / 1e9, "peak_Gops": sfu_peak / 1e9, "frac": sfu_ach / sfu_peak,
                       "tensor_ceiling_frac": ceiling,
                       "note": ("SFU-bound at this head dim: the tensor fraction cannot exceed tensor_ceiling_frac"
                                if ceiling < 1.0 else "tensor-bound at this head dim (the SFU ceiling is above the "
                                "tensor peak)")}
    total_flops = sum(v[1] for v in stages.values())
    step_tflops = total_flops / (ms / 1000.0) / 1e12
    traffic_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(traffic_path):
        try:
            with open(traffic_path) as f:
                tr = json.load(f).get(args.config, {}).get(tname)
            if tr:
                # dram__bytes_read.sum + dram__bytes_write.sum of one launch (ncu --set full)
                roof["traffic"] = tr["dram_bytes_per_launch"] if isinstance(tr, dict) else tr
                if isinstance(tr, dict):
                    roof["traffic_source"] = tr.get("source")
        except Exception:
            pass

    # ---------------- e2e through the C ABI, pinned host buffers
    pinned = {}
    for k in BATCH_KEYS:
        a = np.ascontiguousarray(batch[k])
        t = torch.empty(a.shape, dtype={np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int64,
                                        np.dtype(np.uint8): torch.uint8}[a.dtype], pin_memory=True)
        t.numpy()[...] = a
        pinned[k] = t.numpy()
    h2d = batch_nbytes(pinned)
    # (1) one synchronous call per step (mtfm_cuda_forward): host layout + H2D +
    #     kernels + D2H back to back
    e2e_times = []
    for i in range(args.e2e_steps + 1):
        barrier()
        t0 = time.perf_counter()
        ra = model.forward_batch(pinned)
        t1 = time.perf_counter()
        if i > 0:
            e2e_times.append(t1 - t0)
    e2e_sync_s = float(np.median(e2e_times))
    d2h = len(ra) * (8 + 4 + 4 + 4 + 4 + 8)
    # (2) the split API with two batch objects used alternately (batch_update /
    #     batch_run / batch_results): step i's host layout + H2D run while step
    #     i-1's kernels execute and step i-1's records come back; every step still
    #     copies its inputs from pinned host memory and reads its records back
    pipe = [model.prepare(pinned), model.prepare(pinned)]
    for pbx in pipe:
        pbx.run()
        pbx.results()
    n_pipe = max(args.e2e_steps, 2)
    barrier()
    t0 = time.perf_counter()
    prev = None
    for i in range(n_pipe):
        cur = pipe[i % 2]
        cur.update(pinned)
        cur.run()
        if prev is not None:
            ra = prev.results()
        prev = cur
    ra = prev.results()
    t1 = time.perf_counter()
    e2e_s = (t1 - t0) / n_pipe
    for pbx in pipe:
        pbx.free()
    if dist is not None:
        t = torch.tensor([e2e_s, e2e_sync_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s, e2e_sync_s = float(t[0].item()), float(t[1].item())
    e2e_value = total_targets / e2e_s

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        threads = os.cpu_count() or 1
        inputs = write_cpu_inputs(batch, wl.schemas, wl.cfg, params, [n for n, _, _ in model.param_specs()])
        cb = cpu_baseline(inputs, threads, args.ref_users, reps=2)
        if cb and "error" not in cb:
            cpu = {"value": cb["targets_per_sec"], "unit": "targets/s", "cores": threads, "kind": "reference",
                   "cpu_model": cpu_model(), "build": cb["build"],
                   "sample": f"first {cb['users']} users of this batch ({cb['targets']} targets, same bytes and "
                             f"weights, best of 2 reps), reference Model<float>::forward_sample on std::thread "
                             f"workers"}
        else:
            cpu = {"value": None, "unit": "targets/s", "cores": threads, "kind": "reference",
                   "sample": f"unavailable: {cb}"}
    clocks = clk.summary()
    line = {
        "metric": "scored targets/sec (device-timed)", "value": value, "unit": "targets/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"MTFM-{args.config}", "users_per_gpu": int(len(batch["user_id"])),
                   "targets_per_rank": rank_targets,
                   "tokens_per_gpu": n_tokens, "targets_per_gpu": n_targets,
                   "layers": f"({wl.cfg.hta.target_layers}:{wl.cfg.hta.full_layers})x{wl.cfg.hta.blocks}",
                   "d_model": wl.cfg.hta.d_model, "heads": wl.cfg.hta.heads, "kv_heads": wl.cfg.hta.kv_heads,
                   "parallelism": f"users sharded, {world} GPU(s), no data-path collective",
                   **({"pruned_2_4": True, "sparse_mma": sparse_active} if args.prune else {}),
                   "l2": "inputs/activations > L2 (X alone is %.0f MB)" % (n_tokens * wl.cfg.hta.d_model * 4 / 1e6)},
        "e2e": {"value": e2e_value, "unit": "targets/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_s * 1000, "api": "batch_update/batch_run/batch_results, two batches in flight",
                "sync_call": {"value": total_targets / e2e_sync_s, "ms_per_step": e2e_sync_s * 1000,
                              "api": "mtfm_cuda_forward, one call per step"}},
        "gpu_launches": launches_per_step * args.steps,
        "roofline": roof,
        "step_tflops": step_tflops,
        "step_frac_of_bf16_peak": step_tflops / tflops,
        "stages_ms": {k: round(v[0], 4) for k, v in sorted(stages.items(), key=lambda kv: -kv[1][0])},
        "cpu_baseline": cpu,
        "clocks": clocks,
    }
    print(json.dumps(line))
    if args.profile_json:
        with open(args.profile_json, "w") as f:
            json.dump({"stages": stages, "prof": prof}, f, indent=1)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
