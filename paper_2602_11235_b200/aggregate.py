"""User-level sample aggregation on the GPU (mtfm_cuda_aggregate_users).

    aggregate_users(scenario_ids, stream, store)  ~ aggregate_users (datagen.cpp:171-216)

stream : dict of the exposure stream in arrival order — user_id[n] (int64),
         scenario[n], ts[n] (int64), feat_off[n+1], blk[3n] (user / cross /
         item id counts), feats (ids); pack_stream() builds it from
         (user_id, Exposure) pairs.
store  : the shared H/R store (std::map<int64_t, UserContext>) as a packed
         batch without exposures, users in ascending id; pack_store() builds it.
Returns (packed batch of the aggregated UserSamples, exp_src, report):
exp_src[j] is the stream index of output exposure j (labels stay host data).
Unknown scenario / user raise IntegrityError like the reference.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import abi
from .schema import BATCH_DTYPES, BATCH_KEYS, normalize_batch, pack_samples

STREAM_DTYPES = {"user_id": np.int64, "scenario": np.int32, "ts": np.int64, "feat_off": np.int32, "blk": np.int32,
                 "feats": np.int32}


def pack_stream(pairs) -> dict:
    """[(user_id, Exposure)] -> stream arrays."""
    uid, sc, ts, foff, blk, feats = [], [], [], [0], [], []
    for u, e in pairs:
        uid.append(u)
        sc.append(e.scenario_id)
        ts.append(e.timestamp)
        blk.extend([len(e.user_features), len(e.cross_features), len(e.item_features)])
        feats.extend(e.user_features)
        feats.extend(e.cross_features)
        feats.extend(e.item_features)
        foff.append(len(feats))
    raw = dict(user_id=uid, scenario=sc, ts=ts, feat_off=foff, blk=blk, feats=feats)
    return {k: np.ascontiguousarray(np.asarray(v, dtype=STREAM_DTYPES[k])) for k, v in raw.items()}


def pack_store(store: dict) -> dict:
    """{user_id: (historical_sequences, realtime_sequences)} -> packed batch (ascending ids)."""
    from .schema import UserSample
    return pack_samples([UserSample(u, list(h), list(r), []) for u, (h, r) in sorted(store.items())])


def aggregate_users(scenario_ids, stream: dict, store: dict, device: int = 0):
    L = abi.lib()
    sid = np.ascontiguousarray(np.asarray(sorted(scenario_ids), dtype=np.int32))
    st = {k: np.ascontiguousarray(np.asarray(stream[k], dtype=STREAM_DTYPES[k])) for k in STREAM_DTYPES}
    n = len(st["user_id"])
    if len(st["feat_off"]) != n + 1 or len(st["blk"]) != 3 * n or len(st["scenario"]) != n or len(st["ts"]) != n:
        raise abi.DimensionError("aggregate_users: stream arrays disagree in length")
    sv = abi.ExposureStream(n, len(st["feats"]), *(abi.ptr(st[k]) for k in STREAM_DTYPES))
    sb = normalize_batch(store)
    pb = abi.PackedBatch(len(sb["user_id"]), len(sb["seq_kind"]), len(sb["ev_ts"]), len(sb["exp_ts"]),
                         len(sb["ev_feats"]), len(sb["exp_feats"]), *(abi.ptr(sb[k]) for k in BATCH_KEYS))
    h = C.c_void_p()
    rep = abi.AggregationReport()
    abi.check(L.mtfm_cuda_aggregate_users(device, abi.ptr(sid), len(sid), C.byref(sv), C.byref(pb), C.byref(h),
                                          C.byref(rep)))
    try:
        sz = abi.PackedSizes()
        abi.check(L.mtfm_cuda_aggregate_sizes(h, C.byref(sz)))
        U, S, E, X = sz.n_users, sz.n_seqs, sz.n_events, sz.n_exposures
        shapes = dict(user_id=U, seq_off=U + 1, seq_kind=S, seq_schema=S, ev_off=S + 1, ev_ts=E, ev_feat_off=E + 1,
                      ev_feats=sz.n_ev_feats, exp_off=U + 1, exp_scenario=X, exp_ts=X, exp_feat_off=X + 1,
                      exp_blk=3 * X, exp_feats=sz.n_exp_feats)
        out = {k: np.zeros(shapes[k], BATCH_DTYPES[k]) for k in BATCH_KEYS}
        src = np.zeros(X, np.int32)
        bufs = abi.PackedBuffers(*(abi.ptr(out[k]) for k in BATCH_KEYS), abi.ptr(src))
        abi.check(L.mtfm_cuda_aggregate_fetch(h, C.byref(bufs)))
    finally:
        L.mtfm_cuda_aggregate_free(h)
    report = dict(n_exposure_records=rep.n_exposure_records, n_user_samples=rep.n_user_samples,
                  compression_ratio=rep.compression_ratio)
    return out, src, report
