"""User sharding across GPUs: users are independent, so a batch
is partitioned across ranks with no collective on the data path.

shard_plan(batch, world, cfg=...)  greedy LPT over each user's algorithmic
                           MACs under the model config (projections,
                           mask-aware attention, tokenizer): returns a list
                           of user-index arrays.
take_users(batch, users)   re-packs a subset of users into a new packed batch
                           (include/mtfm_cuda.h layout), preserving order.
"""
from __future__ import annotations

import heapq

import numpy as np

from .schema import normalize_batch


def visible_keys(batch):
    """Per user (sum of c_i over context rows, sum over T rows): the mask-aware
    visible-key counts of mask.hpp:35-40 in the prefix form (row i sees the L_H
    history keys, the realtime keys strictly older than it, and itself if it is
    a T token)."""
    b = normalize_batch(batch)
    U = len(b["user_id"])
    c_ctx = np.zeros(U, np.float64)
    c_t = np.zeros(U, np.float64)
    for u in range(U):
        h, r = [], []
        for q in range(b["seq_off"][u], b["seq_off"][u + 1]):
            ts = b["ev_ts"][b["ev_off"][q]:b["ev_off"][q + 1]]
            (r if b["seq_kind"][q] else h).append(ts)
        h = np.concatenate(h) if h else np.zeros(0, np.int64)
        r = np.sort(np.concatenate(r)) if r else np.zeros(0, np.int64)
        t = b["exp_ts"][b["exp_off"][u]:b["exp_off"][u + 1]]
        lh = len(h)
        c_ctx[u] = lh * (lh + len(r)) + np.searchsorted(r, h, "left").sum() + np.searchsorted(r, r, "left").sum()
        c_t[u] = len(t) * (lh + 1) + np.searchsorted(r, t, "left").sum()
    return c_ctx, c_t


def user_costs(batch, cfg=None):
    """Algorithmic MACs per user: projections per complexity.hpp:54-64,
    mask-aware attention 2*hd*sum(c_i) per layer, tokenizer MLPs. cfg is the
    ModelConfig (default: MTFM-small)."""
    if cfg is None:
        from .schema import HTAConfig, ModelConfig
        cfg = ModelConfig(HTAConfig(d_model=256, blocks=1, target_layers=3, full_layers=1, heads=8, kv_heads=2),
                          d_expert=256)
    h = cfg.hta
    d = h.d_model
    dh = d // h.heads
    hd, gd = h.heads * dh, h.kv_heads * dh
    b = normalize_batch(batch)
    U = len(b["user_id"])
    ev0 = b["ev_off"][b["seq_off"][:-1]] if len(b["ev_off"]) > 1 else np.zeros(U, np.int64)
    ev1 = b["ev_off"][b["seq_off"][1:]] if len(b["ev_off"]) > 1 else np.zeros(U, np.int64)
    n_ctx = (ev1 - ev0).astype(np.float64)
    n_t = np.diff(b["exp_off"]).astype(np.float64)
    n = n_ctx + n_t
    c_ctx, c_t = visible_keys(b)
    full = n * d * (2 * hd + 2 * gd) + n * hd * d + 2.0 * hd * (c_ctx + c_t)
    tgt = n_t * d * 2 * hd + n * d * 2 * gd + n_t * hd * d + 2.0 * hd * c_t
    tok = n * (3 * cfg.d_emb * 2 * d + 2 * d * d)
    return h.blocks * (h.full_layers * full + h.target_layers * tgt) + tok + 1.0


def shard_plan(batch, world, costs=None, cfg=None):
    """Greedy longest-processing-time assignment; each shard keeps batch order."""
    if costs is None:
        costs = user_costs(batch, cfg)
    order = np.argsort(-costs, kind="stable")
    heap = [(0.0, r) for r in range(world)]
    owner = np.empty(len(costs), np.int64)
    for u in order:
        load, r = heapq.heappop(heap)
        owner[u] = r
        heapq.heappush(heap, (load + float(costs[u]), r))
    return [np.nonzero(owner == r)[0] for r in range(world)]


def take_users(batch, users):
    """Packed sub-batch of the given users (in the given order)."""
    b = normalize_batch(batch)
    users = np.asarray(users, np.int64)
    seq_off, ev_off, exp_off = b["seq_off"], b["ev_off"], b["exp_off"]
    ev_fo, ex_fo = b["ev_feat_off"], b["exp_feat_off"]
    seqs = [np.arange(seq_off[u], seq_off[u + 1]) for u in users]
    seq_idx = np.concatenate(seqs) if seqs else np.zeros(0, np.int64)
    n_seq = np.array([len(s) for s in seqs], np.int64)
    ev_len = (ev_off[seq_idx + 1] - ev_off[seq_idx]).astype(np.int64)
    evs = np.concatenate([np.arange(ev_off[s], ev_off[s + 1]) for s in seq_idx]) if len(seq_idx) else \
        np.zeros(0, np.int64)
    xs = np.concatenate([np.arange(exp_off[u], exp_off[u + 1]) for u in users]) if len(users) else \
        np.zeros(0, np.int64)
    n_x = np.array([exp_off[u + 1] - exp_off[u] for u in users], np.int64)

    def cat_ranges(off, idx):
        parts = [np.arange(off[i], off[i + 1]) for i in idx]
        return np.concatenate(parts) if parts else np.zeros(0, np.int64)

    ev_flen = (ev_fo[evs + 1] - ev_fo[evs]).astype(np.int64) if len(evs) else np.zeros(0, np.int64)
    ex_flen = (ex_fo[xs + 1] - ex_fo[xs]).astype(np.int64) if len(xs) else np.zeros(0, np.int64)
    out = dict(
        user_id=b["user_id"][users],
        seq_off=np.concatenate([[0], np.cumsum(n_seq)]),
        seq_kind=b["seq_kind"][seq_idx],
        seq_schema=b["seq_schema"][seq_idx],
        ev_off=np.concatenate([[0], np.cumsum(ev_len)]),
        ev_ts=b["ev_ts"][evs],
        ev_feat_off=np.concatenate([[0], np.cumsum(ev_flen)]),
        ev_feats=b["ev_feats"][cat_ranges(ev_fo, evs)],
        exp_off=np.concatenate([[0], np.cumsum(n_x)]),
        exp_scenario=b["exp_scenario"][xs],
        exp_ts=b["exp_ts"][xs],
        exp_feat_off=np.concatenate([[0], np.cumsum(ex_flen)]),
        exp_blk=b["exp_blk"].reshape(-1, 3)[xs].reshape(-1),
        exp_feats=b["exp_feats"][cat_ranges(ex_fo, xs)],
    )
    return normalize_batch(out)
