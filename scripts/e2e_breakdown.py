"""Host-side breakdown of one end-to-end forward (normalize, pack, count, C forward)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import torch
from paper_2602_11235_b200 import Model, datagen, abi
from paper_2602_11235_b200.schema import normalize_batch

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
for _ in range(3):
    model.forward_batch(pinned)
T = {}
def tic(k, t0):
    T.setdefault(k, []).append(time.perf_counter() - t0)
for _ in range(10):
    t0 = time.perf_counter(); b = normalize_batch(pinned); tic("normalize", t0)
    t0 = time.perf_counter(); pb = model._packed(b); tic("pack", t0)
    t0 = time.perf_counter(); n = int(abi.lib().mtfm_cuda_count_records(model._h, C.byref(pb))); tic("count", t0)
    t0 = time.perf_counter(); out, rec = model._record_buffers(n); tic("recbuf", t0)
    t0 = time.perf_counter(); abi.check(abi.lib().mtfm_cuda_forward(model._h, C.byref(pb), -1, C.byref(rec))); tic("forward", t0)
    t0 = time.perf_counter(); h = C.c_void_p(); abi.check(abi.lib().mtfm_cuda_batch_prepare(model._h, C.byref(pb), -1, C.byref(h))); torch.cuda.synchronize(); tic("prepare+h2d", t0)
    t0 = time.perf_counter(); abi.check(abi.lib().mtfm_cuda_batch_run(model._h, h)); tic("run_enqueue", t0)
    t0 = time.perf_counter(); abi.check(abi.lib().mtfm_cuda_batch_results(model._h, h, C.byref(rec))); tic("results(wait+d2h)", t0)
    abi.lib().mtfm_cuda_batch_free(h)
for k, v in T.items():
    print(f"{k:20s} median {np.median(v)*1e3:8.3f} ms")
