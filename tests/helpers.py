"""Shared test helpers: conversions between the package's schema objects and
the oracle's, and record comparison."""
import numpy as np

import mtfm_oracle as O
from paper_2602_11235_b200.schema import (HTAConfig, ModelConfig, ScenarioSchema, SchemaSet, SequenceSchema)


def to_oracle(sch: SchemaSet, cfg: ModelConfig):
    osch = O.Schemas([(s.seq_id, list(s.feature_vocabs)) for s in sch.hist],
                     [(s.seq_id, list(s.feature_vocabs)) for s in sch.rt],
                     [(s.scenario_id, list(s.user_feature_vocabs), list(s.cross_feature_vocabs),
                       list(s.item_feature_vocabs), list(s.tasks)) for s in sch.scenarios])
    h = cfg.hta
    ocfg = O.Config(d_model=h.d_model, blocks=h.blocks, target_layers=h.target_layers, full_layers=h.full_layers,
                    heads=h.heads, kv_heads=h.kv_heads, norm=h.norm, eps=h.eps, d_emb=cfg.d_emb,
                    experts=cfg.experts, d_expert=cfg.d_expert)
    return osch, ocfg


def from_oracle(osch: O.Schemas, ocfg: O.Config):
    sch = SchemaSet([SequenceSchema(i, list(v)) for i, v in osch.hist],
                    [SequenceSchema(i, list(v)) for i, v in osch.rt],
                    [ScenarioSchema(i, list(u), list(c), list(x), list(t)) for i, u, c, x, t in osch.scen])
    cfg = ModelConfig(HTAConfig(d_model=ocfg.d_model, blocks=ocfg.blocks, target_layers=ocfg.target_layers,
                                full_layers=ocfg.full_layers, heads=ocfg.heads, kv_heads=ocfg.kv_heads,
                                norm=ocfg.norm, eps=ocfg.eps),
                      d_emb=ocfg.d_emb, experts=ocfg.experts, d_expert=ocfg.d_expert)
    return sch, cfg


def oracle_records(osch, ocfg, params, batch, dtype=np.float64):
    recs = O.Oracle(osch, ocfg, params, dtype).forward_batch(batch)
    keys = np.array([r[:4] for r in recs], dtype=np.int64).reshape(-1, 4)
    z = np.array([r[4] for r in recs], dtype=np.float64)
    p = np.array([r[5] for r in recs], dtype=np.float64)
    return keys, z, p


def check_floor(name):
    """Floor of the fp32 check metric for a golden fixture: 1e-2 for the
    default-initialised fixtures (|z| < 0.15), 1.0 for the jittered ones whose
    logits are O(1) (median |z| 1.1-1.8): there the reference's own Model<float>
    misses 1e-4 against its f64 path at a 0.1 floor (1.4e-4 on base_j) and meets
    it at 1.0 (2.4e-5), so the floor is the logit scale, and errors on logits below
    1 are held to 1e-4 absolute."""
    return 1.0 if name.endswith("_j") else 1e-2


def rel_err(z, ref, floor=1e-2):
    """max |z - ref| / max(|ref|, floor) — the fp32 check-mode metric.

    The floor is 1e-2, not 1e-3: logits of these randomly initialised models
    sit near zero (|z| < 0.15) and the reference's own f32 path
    (Model<float>) misses 1e-4 against its f64 path under a 1e-3 floor
    (1.23e-4 on small4) while meeting it with margin under 1e-2 (1.8e-5); see
    tests/test_oracle_golden.py::test_reference_f32_meets_check_metric."""
    if len(ref) == 0:
        return 0.0
    return float(np.max(np.abs(z - ref) / np.maximum(np.abs(ref), floor)))
