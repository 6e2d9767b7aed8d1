"""Dataset ingestion: the reference's line-delimited dataset file
(dataset_io.cpp:110-221) -> page-locked packed jagged batches, parsed natively
by worker threads (mtfm_dataset_load), then scored with the upload of chunk
i+1 overlapping the kernels of chunk i.

    ds = load_dataset(path, threads=0, chunk_users=1024)  ~ load_dataset
    ds.schemas                  SchemaSet of the header
    ds.chunk(i) -> (batch, labels)  zero-copy views of the pinned arrays
    score_dataset(model, ds)    every chunk through the split C API, two batch
                                objects in flight; records with their labels
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import abi
from .schema import BATCH_DTYPES, BATCH_KEYS, ScenarioSchema, SchemaSet, SequenceSchema


def _view(ptr, n, dtype):
    if n == 0 or not ptr:
        return np.zeros(0, dtype)
    buf = (C.c_char * (n * np.dtype(dtype).itemsize)).from_address(ptr)
    return np.frombuffer(buf, dtype=dtype, count=n)


class Dataset:
    def __init__(self, path, threads=0, chunk_users=1024):
        L = abi.lib()
        h = C.c_void_p()
        abi.check(L.mtfm_dataset_load(str(path).encode(), int(threads), int(chunk_users), C.byref(h)))
        self._h = h
        info = abi.DatasetInfo()
        abi.check(L.mtfm_dataset_info(h, C.byref(info)))
        self.format_version, self.n_users, self.n_chunks, self.max_tasks = (
            info.format_version, info.n_users, info.n_chunks, info.max_tasks)
        sd = abi.SchemaDesc()
        abi.check(L.mtfm_dataset_schema_desc(h, C.byref(sd)))
        p = 0
        hist = []
        for i in range(sd.n_hist):
            n = sd.hist_nslots[i]
            hist.append(SequenceSchema(sd.hist_ids[i], [sd.hist_vocabs[p + k] for k in range(n)]))
            p += n
        p = 0
        rt = []
        for i in range(sd.n_rt):
            n = sd.rt_nslots[i]
            rt.append(SequenceSchema(sd.rt_ids[i], [sd.rt_vocabs[p + k] for k in range(n)]))
            p += n
        sc, p, t = [], 0, 0
        for i in range(sd.n_scen):
            nu, nc, ni = sd.scen_nu[i], sd.scen_nc[i], sd.scen_ni[i]
            v = [sd.scen_vocabs[p + k] for k in range(nu + nc + ni)]
            p += nu + nc + ni
            tasks = [sd.task_names[t + k].decode() for k in range(sd.scen_ntasks[i])]
            t += sd.scen_ntasks[i]
            sc.append(ScenarioSchema(sd.scen_ids[i], v[:nu], v[nu:nu + nc], v[nu + nc:], tasks))
        self.schemas = SchemaSet(hist, rt, sc)

    def chunk(self, i):
        """(packed batch dict, labels [n_exposures][max_tasks]) — views into pinned memory."""
        pb = abi.PackedBatch()
        lab = C.POINTER(C.c_int32)()
        abi.check(abi.lib().mtfm_dataset_chunk(self._h, int(i), C.byref(pb), C.byref(lab)))
        U, S, E, X = pb.n_users, pb.n_seqs, pb.n_events, pb.n_exposures
        n = dict(user_id=U, seq_off=U + 1, seq_kind=S, seq_schema=S, ev_off=S + 1, ev_ts=E, ev_feat_off=E + 1,
                 ev_feats=pb.n_ev_feats, exp_off=U + 1, exp_scenario=X, exp_ts=X, exp_feat_off=X + 1,
                 exp_blk=3 * X, exp_feats=pb.n_exp_feats)
        b = {k: _view(getattr(pb, k), n[k], BATCH_DTYPES[k]) for k in BATCH_KEYS}
        labels = _view(C.cast(lab, C.c_void_p).value, X * self.max_tasks, np.int32).reshape(X, self.max_tasks)
        return b, labels

    def close(self):
        if getattr(self, "_h", None):
            abi.lib().mtfm_dataset_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def load_dataset(path, threads=0, chunk_users=1024) -> Dataset:
    return Dataset(path, threads, chunk_users)


def score_dataset(model, ds: Dataset, only_scenario=-1):
    """Every chunk through batch_update / batch_run / batch_results with two batch
    objects used alternately: chunk i+1's H2D (from the pinned chunk arrays) and
    host layout run while chunk i's kernels execute. Returns per chunk
    (RecordArrays, labels per record)."""
    out = []
    if ds.n_chunks == 0:
        return out
    pipe = []
    prev = None
    ntasks = {sid: len(t) for sid, t in model._tasks.items()}
    if only_scenario >= 0:
        ntasks = {sid: n for sid, n in ntasks.items() if sid == only_scenario}
    for i in range(ds.n_chunks):
        b, labels = ds.chunk(i)
        if len(pipe) < 2:
            pipe.append(model.prepare(b, only_scenario))
            cur = pipe[-1]
        else:
            cur = pipe[i % 2]
            cur.update(b, only_scenario)
        cur.run()
        if prev is not None:
            out.append(_with_labels(prev))
        prev = (cur, labels, ntasks)
    out.append(_with_labels(prev))
    for p in pipe:
        p.free()
    return out


def _with_labels(item):
    pb, labels, ntasks = item
    ra = pb.results()
    b = pb.batch
    # records are user-major in batch order: user of each record, then its exposure row
    per_x = np.array([ntasks.get(int(sc), 0) for sc in b["exp_scenario"]], np.int64)
    per_u = np.add.reduceat(per_x, b["exp_off"][:-1]) if len(per_x) else np.zeros(len(b["user_id"]), np.int64)
    per_u = np.where(np.diff(b["exp_off"]) > 0, per_u, 0)
    u = np.repeat(np.arange(len(b["user_id"])), per_u)
    x = b["exp_off"][u] + ra.exposure_index
    lab = labels[x, ra.task_index] if len(ra) else np.zeros(0, np.int32)
    return ra, lab
