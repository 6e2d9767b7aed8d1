"""Host mirror of the reference data model (proj/include/mtfm/schema.hpp,
model_config.hpp) and the packed jagged batch of include/mtfm_cuda.h.

Names follow the reference: SequenceSchema, ScenarioSchema, SchemaSet,
HTAConfig, ModelConfig, BehaviorEvent, SequenceRecord, Exposure, UserSample,
InferenceRequest, PredictionRecord.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class SequenceSchema:  # schema.hpp:18-24
    seq_id: int
    feature_vocabs: list


@dataclass
class ScenarioSchema:  # schema.hpp:27-41
    scenario_id: int
    user_feature_vocabs: list
    cross_feature_vocabs: list
    item_feature_vocabs: list
    tasks: list


@dataclass
class SchemaSet:  # model.hpp:117-136
    hist: list
    rt: list
    scenarios: list

    def tasks_by_scenario(self):
        return {s.scenario_id: list(s.tasks) for s in self.scenarios}

    def scenario(self, sid):
        for s in self.scenarios:
            if s.scenario_id == sid:
                return s
        return None


@dataclass
class HTAConfig:  # model_config.hpp:39-74
    d_model: int = 64
    blocks: int = 4
    target_layers: int = 3
    full_layers: int = 1
    heads: int = 4
    kv_heads: int = 2
    norm: str = "valid"
    eps: float = 1e-6

    @property
    def head_dim(self):
        return self.d_model // self.heads


@dataclass
class ModelConfig:  # model_config.hpp:76-88
    hta: HTAConfig = field(default_factory=HTAConfig)
    d_emb: int = 16
    experts: int = 4
    d_expert: int = 64


@dataclass
class BehaviorEvent:  # schema.hpp:45-50
    item_features: list
    timestamp: int


@dataclass
class SequenceRecord:  # schema.hpp:52-57
    seq_schema_id: int
    events: list


@dataclass
class Exposure:  # schema.hpp:60-69
    scenario_id: int
    user_features: list
    cross_features: list
    item_features: list
    timestamp: int
    labels: dict = field(default_factory=dict)


@dataclass
class UserSample:  # schema.hpp:72-80
    user_id: int
    historical_sequences: list
    realtime_sequences: list
    exposures: list


@dataclass
class Candidate:  # schema.hpp:83-89
    user_features: list
    cross_features: list
    item_features: list


@dataclass
class InferenceRequest:  # schema.hpp:92-99
    user_id: int
    scenario_id: int
    timestamp: int
    historical_sequences: list
    realtime_sequences: list
    candidates: list


@dataclass
class PredictionRecord:  # records.hpp:10-19
    user_id: int
    scenario_id: int
    exposure_index: int
    task: str
    probability: float
    label: int = -1


def sample_view_of_request(r: InferenceRequest) -> UserSample:
    """tokenizer.hpp:138-153: candidates share the request timestamp, no labels."""
    return UserSample(r.user_id, list(r.historical_sequences), list(r.realtime_sequences),
                      [Exposure(r.scenario_id, c.user_features, c.cross_features, c.item_features, r.timestamp)
                       for c in r.candidates])


BATCH_KEYS = ("user_id", "seq_off", "seq_kind", "seq_schema", "ev_off", "ev_ts", "ev_feat_off", "ev_feats",
              "exp_off", "exp_scenario", "exp_ts", "exp_feat_off", "exp_blk", "exp_feats")
BATCH_DTYPES = {"user_id": np.int64, "seq_off": np.int32, "seq_kind": np.uint8, "seq_schema": np.int32,
                "ev_off": np.int32, "ev_ts": np.int64, "ev_feat_off": np.int32, "ev_feats": np.int32,
                "exp_off": np.int32, "exp_scenario": np.int32, "exp_ts": np.int64, "exp_feat_off": np.int32,
                "exp_blk": np.int32, "exp_feats": np.int32}


def pack_samples(samples) -> dict:
    """Flattens UserSamples into the packed jagged batch (no sorting)."""
    user_id, seq_off, seq_kind, seq_schema = [], [0], [], []
    ev_off, ev_ts, ev_feat_off, ev_feats = [0], [], [0], []
    exp_off, exp_scen, exp_ts, exp_feat_off, exp_blk, exp_feats = [0], [], [], [0], [], []
    for s in samples:
        user_id.append(s.user_id)
        for kind, seqs in ((0, s.historical_sequences), (1, s.realtime_sequences)):
            for rec in seqs:
                seq_kind.append(kind)
                seq_schema.append(rec.seq_schema_id)
                for ev in rec.events:
                    ev_ts.append(ev.timestamp)
                    ev_feats.extend(ev.item_features)
                    ev_feat_off.append(len(ev_feats))
                ev_off.append(len(ev_ts))
        seq_off.append(len(seq_kind))
        for e in s.exposures:
            exp_scen.append(e.scenario_id)
            exp_ts.append(e.timestamp)
            exp_blk.extend([len(e.user_features), len(e.cross_features), len(e.item_features)])
            exp_feats.extend(e.user_features)
            exp_feats.extend(e.cross_features)
            exp_feats.extend(e.item_features)
            exp_feat_off.append(len(exp_feats))
        exp_off.append(len(exp_scen))
    raw = dict(user_id=user_id, seq_off=seq_off, seq_kind=seq_kind, seq_schema=seq_schema, ev_off=ev_off,
               ev_ts=ev_ts, ev_feat_off=ev_feat_off, ev_feats=ev_feats, exp_off=exp_off, exp_scenario=exp_scen,
               exp_ts=exp_ts, exp_feat_off=exp_feat_off, exp_blk=exp_blk, exp_feats=exp_feats)
    return {k: np.ascontiguousarray(np.asarray(v, dtype=BATCH_DTYPES[k])) for k, v in raw.items()}


def normalize_batch(batch: dict) -> dict:
    return {k: np.ascontiguousarray(np.asarray(batch[k], dtype=BATCH_DTYPES[k])) for k in BATCH_KEYS}


def batch_nbytes(batch: dict) -> int:
    return int(sum(np.asarray(batch[k]).nbytes for k in BATCH_KEYS))


def param_specs(schemas: SchemaSet, cfg: ModelConfig):
    """[(name, rows, cols)] in Model::register_params order (model.hpp:377-463);
    host-side, no device needed. The library registers the same list
    (mtfm_cuda_param_name)."""
    h = cfg.hta
    d, de = h.d_model, cfg.d_emb
    dh = d // h.heads
    hd, gd = h.heads * dh, h.kv_heads * dh
    out = []
    srcs = ([("h", s.seq_id, [s.feature_vocabs]) for s in schemas.hist] +
            [("r", s.seq_id, [s.feature_vocabs]) for s in schemas.rt] +
            [("s", s.scenario_id, [s.user_feature_vocabs, s.cross_feature_vocabs, s.item_feature_vocabs])
             for s in schemas.scenarios])
    for kind, sid, blocks in srcs:
        base = f"tok/{kind}{sid}"
        k_in = 0
        if kind != "s":
            for k, v in enumerate(blocks[0]):
                out.append((f"{base}/emb{k}", v, de))
                k_in += de
        else:
            for pre, vs in zip(("emb_u", "emb_c", "emb_i"), blocks):
                for k, v in enumerate(vs):
                    out.append((f"{base}/{pre}{k}", v, de))
                    k_in += de
        out += [(f"{base}/mlp_w1", k_in, 2 * d), (f"{base}/mlp_b1", 1, 2 * d), (f"{base}/mlp_w2", 2 * d, d),
                (f"{base}/mlp_b2", 1, d)]
    keys = [("h", s.seq_id, False) for s in schemas.hist] + [("r", s.seq_id, False) for s in schemas.rt] + \
        [("t", s.scenario_id, True) for s in schemas.scenarios]
    for b in range(h.blocks):
        for l in range(h.target_layers + h.full_layers):
            tgt = l < h.target_layers
            base = f"hta/b{b}/l{l}"
            if tgt:
                out += [(f"{base}/fuq_w", d, 2 * hd), (f"{base}/fuq_b", 1, 2 * hd), (f"{base}/fkv_w", d, 2 * gd),
                        (f"{base}/fkv_b", 1, 2 * gd)]
            else:
                out += [(f"{base}/f1_w", d, 2 * hd + 2 * gd), (f"{base}/f1_b", 1, 2 * hd + 2 * gd)]
            out += [(f"{base}/f2_w", hd, d), (f"{base}/f2_b", 1, d)]
            for k, sid, scen in keys:
                out += [(f"{base}/gln1/{k}{sid}/gain", 1, d), (f"{base}/gln1/{k}{sid}/bias", 1, d)]
                if not tgt or scen:
                    out += [(f"{base}/gln2/{k}{sid}/gain", 1, hd), (f"{base}/gln2/{k}{sid}/bias", 1, hd)]
    for e in range(cfg.experts):
        out += [(f"head/expert{e}_w", d, cfg.d_expert), (f"head/expert{e}_b", 1, cfg.d_expert)]
    for s in schemas.scenarios:
        for t in s.tasks:
            base = f"head/s{s.scenario_id}/{t}"
            out += [(f"{base}/gate_w", d, cfg.experts), (f"{base}/gate_b", 1, cfg.experts),
                    (f"{base}/tower_w", cfg.d_expert, 1), (f"{base}/tower_b", 1, 1)]
    return out
