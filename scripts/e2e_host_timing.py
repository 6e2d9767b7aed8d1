"""Host-side cost of one pipelined e2e step at MTFM-small (where the 3 % e2e gap goes):
times batch_update (layout + H2D enqueue), batch_run (enqueue) and batch_results."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch  # noqa: E402

from paper_2602_11235_b200 import Model, datagen  # noqa: E402
from paper_2602_11235_b200.schema import BATCH_KEYS  # noqa: E402

wl = datagen.WORKLOADS["small"]()
b = datagen.generate(wl)
m = Model(wl.schemas, wl.cfg, precision="bf16")
m.set_params(datagen.random_params(m.param_specs(), seed=7))
pinned = {}
for k in BATCH_KEYS:
    a = np.ascontiguousarray(b[k])
    t = torch.empty(a.shape, dtype={np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int64,
                                    np.dtype(np.uint8): torch.uint8}[a.dtype], pin_memory=True)
    t.numpy()[...] = a
    pinned[k] = t.numpy()
pipe = [m.prepare(pinned), m.prepare(pinned)]
for p in pipe:
    p.run()
    p.results()
tu, tr, tq = [], [], []
prev = None
t_all = time.perf_counter()
for i in range(40):
    cur = pipe[i % 2]
    t0 = time.perf_counter()
    cur.update(pinned)
    t1 = time.perf_counter()
    cur.run()
    t2 = time.perf_counter()
    if prev is not None:
        prev.results()
    t3 = time.perf_counter()
    tu.append(t1 - t0)
    tr.append(t2 - t1)
    tq.append(t3 - t2)
    prev = cur
prev.results()
t_all = time.perf_counter() - t_all
print(f"per step: update {1e3 * np.median(tu):.3f} ms, run {1e3 * np.median(tr):.3f} ms, results (incl. wait) "
      f"{1e3 * np.median(tq):.3f} ms; wall {1e3 * t_all / 40:.3f} ms/step")
