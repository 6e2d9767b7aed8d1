"""Host-side timing of the pipelined split API loop used by bench.py's e2e
(update / run / results on two batch objects, MTFM-small)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_11235_b200 import Model, datagen

wl = datagen.WORKLOADS["small"]()
batch = datagen.generate(wl)
model = Model(wl.schemas, wl.cfg, precision="bf16", device=0)
model.set_params(datagen.random_params(model.param_specs(), seed=7))
pinned = {}
for k, a in batch.items():
    a = np.ascontiguousarray(a)
    t = torch.empty(a.shape, dtype={np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int64,
                                    np.dtype(np.uint8): torch.uint8}[a.dtype], pin_memory=True)
    t.numpy()[...] = a
    pinned[k] = t.numpy()
pipe = [model.prepare(pinned), model.prepare(pinned)]
for p in pipe:
    p.run(); p.results()
T = {"update": [], "run": [], "results": [], "step": []}
prev = None
n = 40
t_all = time.perf_counter()
for i in range(n):
    cur = pipe[i % 2]
    t0 = time.perf_counter(); cur.update(pinned); t1 = time.perf_counter(); cur.run(); t2 = time.perf_counter()
    if prev is not None:
        prev.results()
    t3 = time.perf_counter()
    prev = cur
    T["update"].append(t1 - t0); T["run"].append(t2 - t1); T["results"].append(t3 - t2); T["step"].append(t3 - t0)
prev.results()
print("per step %.3f ms" % ((time.perf_counter() - t_all) / n * 1e3))
for k, v in T.items():
    print(f"{k:10s} median {np.median(v)*1e3:7.3f} ms  p90 {np.percentile(v, 90)*1e3:7.3f}")
