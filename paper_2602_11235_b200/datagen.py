"""Synthetic workloads of the BASELINE.json configurations, generated straight
into the packed jagged batch layout (vectorised numpy; seeded).

Schemas follow the reference generator's heterogeneous layout
(proj/src/datagen.cpp:226-251): historical schema i has 2 + i%2 slots with
vocabs item_vocab + 17i + 5j; realtime schemas 2 slots, item_vocab + 23i + 3j;
scenario s has 2 + s%3 user, 1 + (s+1)%2 cross and 2 + (s+2)%3 item slots and
tasks {ctr, ctcvr} (scenario 1: + imd, write). Timestamps use the reference
windows (datagen.cpp:36-40): H in [0, 1000), R in [700, 2000), T in
[1000, 2000); every sequence is time-sorted. Labels are not generated (the
scored forward does not read them).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .schema import HTAConfig, ModelConfig, ScenarioSchema, SchemaSet, SequenceSchema


def make_schemas(n_scenarios=4, n_hist=2, n_rt=1, base_vocab=120, item_vocab=240) -> SchemaSet:
    hist = [SequenceSchema(i, [item_vocab + 17 * i + 5 * j for j in range(2 + i % 2)]) for i in range(n_hist)]
    rt = [SequenceSchema(i, [item_vocab + 23 * i + 3 * j for j in range(2)]) for i in range(n_rt)]
    sc = []
    for s in range(n_scenarios):
        sc.append(ScenarioSchema(
            s,
            [base_vocab + 37 * s + 13 * j for j in range(2 + s % 3)],
            [base_vocab // 2 + 19 * s + 7 * j for j in range(1 + (s + 1) % 2)],
            [item_vocab + 29 * s + 11 * j for j in range(2 + (s + 2) % 3)],
            ["ctr", "ctcvr", "imd", "write"] if s == 1 else ["ctr", "ctcvr"]))
    return SchemaSet(hist, rt, sc)


@dataclass
class Workload:
    name: str
    cfg: ModelConfig
    schemas: SchemaSet
    n_users: int
    hist_len: object      # int, or ("lognormal", median, sigma, lo, hi)
    rt_len: object
    exp_per_scen: object  # int, or ("lognormal", median, sigma, lo, hi) for the per-user total
    seed: int


def _model(d, blocks, K, P, H, G):
    return ModelConfig(HTAConfig(d_model=d, blocks=blocks, target_layers=K, full_layers=P, heads=H, kv_heads=G),
                       d_emb=16, experts=4, d_expert=d)


# BASELINE.json configs (layers -> (K:P)xB with the paper's K=3, P=1).
WORKLOADS = {
    "tiny": lambda: Workload("tiny", _model(64, 1, 1, 1, 4, 2), make_schemas(), 8, 21, 21, 2, 1),
    "small": lambda: Workload("small", _model(256, 1, 3, 1, 8, 2), make_schemas(), 1024, 224, 64, 8, 3),
    "base": lambda: Workload("base", _model(512, 2, 3, 1, 16, 4), make_schemas(), 4096,
                             ("lognormal", 300 / 3, 0.9, 5, 448), ("lognormal", 300 / 3, 0.9, 5, 128),
                             ("lognormal", 16, 0.8, 1, 64), 11),
    "large": lambda: Workload("large", _model(1024, 4, 3, 1, 16, 4), make_schemas(), 1024, 896, 256, 32, 5),
    "paper": lambda: Workload("paper", _model(768, 4, 3, 1, 3, 1), make_schemas(), 256, 896, 256, 32, 7),
    # multi-scenario aggregation sweep (BASELINE configs[4]): 4 scenarios with distinct token
    # schemas, 1-256 targets per user (heavy-tailed), d=256 8Q/2KV; the HTA mix and G=H are
    # varied by the caller (bench.py --mix / --mha)
    "sweep": lambda: Workload("sweep", _model(256, 1, 3, 1, 8, 2), make_schemas(), 1024,
                              ("lognormal", 160, 0.8, 8, 448), ("lognormal", 48, 0.8, 2, 128),
                              ("lognormal", 24, 1.0, 1, 256), 13),
}


def with_mix(wl: Workload, mix=None, mha=False) -> Workload:
    """The workload with another HTA mix "K:P" and/or G = H (multi-head instead of GQA):
    the reference's bench matrix (bench.hpp:40-57) over a BASELINE workload."""
    import dataclasses
    hta = wl.cfg.hta
    if mix:
        k, p = (int(x) for x in mix.split(":"))
        hta = dataclasses.replace(hta, target_layers=k, full_layers=p)
    if mha:
        hta = dataclasses.replace(hta, kv_heads=hta.heads)
    return dataclasses.replace(wl, cfg=dataclasses.replace(wl.cfg, hta=hta))


def _draw_len(rng, spec, n):
    if isinstance(spec, (int, np.integer)):
        return np.full(n, int(spec), np.int64)
    _, med, sig, lo, hi = spec
    v = np.floor(np.exp(rng.normal(math.log(med), sig, n)))
    return np.clip(v, lo, hi).astype(np.int64)


def generate(wl: Workload, n_users=None) -> dict:
    """Packed batch (include/mtfm_cuda.h layout) for a workload."""
    rng = np.random.default_rng(wl.seed)
    U = wl.n_users if n_users is None else n_users
    sch = wl.schemas
    nh, nr, ns = len(sch.hist), len(sch.rt), len(sch.scenarios)
    # per (user, sequence) lengths, user-major, hist then rt
    lens = np.empty((U, nh + nr), np.int64)
    for i in range(nh):
        lens[:, i] = _draw_len(rng, wl.hist_len, U)
    for i in range(nr):
        lens[:, nh + i] = _draw_len(rng, wl.rt_len, U)
    seq_kind = np.tile(np.array([0] * nh + [1] * nr, np.uint8), U)
    seq_schema = np.tile(np.array([s.seq_id for s in sch.hist] + [s.seq_id for s in sch.rt], np.int32), U)
    seq_len = lens.reshape(-1)
    ev_off = np.zeros(len(seq_len) + 1, np.int64)
    np.cumsum(seq_len, out=ev_off[1:])
    n_ev = int(ev_off[-1])
    seq_of_ev = np.repeat(np.arange(len(seq_len)), seq_len)
    kind_of_ev = seq_kind[seq_of_ev]
    lo = np.where(kind_of_ev == 0, 0, 700)
    hi = np.where(kind_of_ev == 0, 1000, 2000)
    ts = lo + (rng.random(n_ev) * (hi - lo)).astype(np.int64)
    # sort timestamps within each sequence
    order = np.lexsort((ts, seq_of_ev))
    ev_ts = ts[order]
    # features: slots per event from its schema
    slots_of_schema = [len(s.feature_vocabs) for s in sch.hist] + [len(s.feature_vocabs) for s in sch.rt]
    vocab_table = [s.feature_vocabs for s in sch.hist] + [s.feature_vocabs for s in sch.rt]
    sidx = np.tile(np.arange(nh + nr), U)[seq_of_ev]
    nslot_ev = np.array(slots_of_schema)[sidx]
    ev_feat_off = np.zeros(n_ev + 1, np.int64)
    np.cumsum(nslot_ev, out=ev_feat_off[1:])
    feats = np.empty(int(ev_feat_off[-1]), np.int32)
    for k in range(nh + nr):
        m = sidx == k
        idx = ev_feat_off[:-1][m]
        for j, v in enumerate(vocab_table[k]):
            feats[idx + j] = rng.integers(0, v, int(m.sum()))
    # exposures
    if isinstance(wl.exp_per_scen, (int, np.integer)):
        cnt = np.full((U, ns), int(wl.exp_per_scen), np.int64)
    else:
        tot = _draw_len(rng, wl.exp_per_scen, U)
        cnt = np.zeros((U, ns), np.int64)
        pick = rng.integers(0, ns, int(tot.sum()))
        np.add.at(cnt, (np.repeat(np.arange(U), tot), pick), 1)
    exp_per_user = cnt.sum(1)
    n_x = int(exp_per_user.sum())
    sp = (np.concatenate([np.repeat(np.arange(ns), cnt[u]) for u in range(U)]) if n_x
          else np.zeros(0, np.int64))
    scen_ids = np.array([s.scenario_id for s in sch.scenarios], np.int32)
    exp_scen = scen_ids[sp]
    exp_ts = 1000 + (rng.random(n_x) * 1000).astype(np.int64)
    blk = np.array([[len(s.user_feature_vocabs), len(s.cross_feature_vocabs), len(s.item_feature_vocabs)]
                    for s in sch.scenarios], np.int32)
    exp_blk = blk[sp]
    nf = exp_blk.sum(1)
    exp_feat_off = np.zeros(n_x + 1, np.int64)
    np.cumsum(nf, out=exp_feat_off[1:])
    efeats = np.empty(int(exp_feat_off[-1]), np.int32)
    for i, s in enumerate(sch.scenarios):
        m = sp == i
        idx = exp_feat_off[:-1][m]
        for j, v in enumerate(s.user_feature_vocabs + s.cross_feature_vocabs + s.item_feature_vocabs):
            efeats[idx + j] = rng.integers(0, v, int(m.sum()))
    seq_off = (np.arange(U + 1, dtype=np.int32) * (nh + nr)).astype(np.int32)
    exp_off = np.zeros(U + 1, np.int64)
    np.cumsum(exp_per_user, out=exp_off[1:])
    return dict(user_id=np.arange(U, dtype=np.int64), seq_off=seq_off, seq_kind=seq_kind,
                seq_schema=seq_schema, ev_off=ev_off.astype(np.int32), ev_ts=ev_ts,
                ev_feat_off=ev_feat_off.astype(np.int32), ev_feats=feats, exp_off=exp_off.astype(np.int32),
                exp_scenario=exp_scen.astype(np.int32), exp_ts=exp_ts, exp_feat_off=exp_feat_off.astype(np.int32),
                exp_blk=exp_blk.reshape(-1).astype(np.int32), exp_feats=efeats)


def random_params(specs, seed=0, scale_bias=0.1, gln_jitter=0.2):
    """Random weights for a list of (name, rows, cols) parameter specs: weights
    uniform(+-1/sqrt(rows)) as Model::build (model.hpp:461-476); biases and
    GLN gain/bias jittered away from 0/1 so every path is exercised."""
    rng = np.random.default_rng(seed)
    P = {}
    for name, r, c in specs:
        if name.endswith("/gain"):
            v = 1.0 + gln_jitter * rng.uniform(-1, 1, (r, c))
        elif name.endswith("/bias") or name.endswith("_b") or name.endswith("/mlp_b1") or name.endswith("/mlp_b2"):
            v = scale_bias * rng.uniform(-1, 1, (r, c))
        elif "/emb" in name:
            v = rng.uniform(-1, 1, (r, c)) / math.sqrt(c)
        else:
            v = rng.uniform(-1, 1, (r, c)) / math.sqrt(r)
        P[name] = v.astype(np.float32)
    return P
