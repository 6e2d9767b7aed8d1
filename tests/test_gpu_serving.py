"""Request-level serving: scenario-subgraph deployment
(extract_subgraph, subgraph.hpp:25-42) and many InferenceRequests scored in one
forward (infer_request, subgraph.hpp:47-62; sample_view_of_request,
tokenizer.hpp:138-153). Needs a B200."""
import re

import numpy as np
import pytest

import mtfm_oracle as O
from golden_util import batch, model
from helpers import from_oracle
from paper_2602_11235_b200 import Model, abi, infer_request, infer_requests
from paper_2602_11235_b200.schema import Candidate, InferenceRequest, SequenceRecord, BehaviorEvent

pytestmark = pytest.mark.gpu


def owner(name):
    """names::owner_scenario (model.hpp:71-87)."""
    for part in name.split("/"):
        if re.fullmatch(r"[st]\d+", part):
            return int(part[1:])
    return -1


def _requests(b, sch, scenario, n):
    """n requests of one scenario built from the fixture users' sequences."""
    sc = sch.scenario(scenario)
    reqs = []
    for k in range(n):
        u = k % len(b["user_id"])
        hist, rt = [], []
        for q in range(b["seq_off"][u], b["seq_off"][u + 1]):
            evs = [BehaviorEvent([int(f) for f in b["ev_feats"][b["ev_feat_off"][e]:b["ev_feat_off"][e + 1]]],
                                 int(b["ev_ts"][e])) for e in range(b["ev_off"][q], b["ev_off"][q + 1])]
            (rt if b["seq_kind"][q] else hist).append(SequenceRecord(int(b["seq_schema"][q]), evs))
        cands = [Candidate([(c * 7 + k + j) % v for j, v in enumerate(sc.user_feature_vocabs)],
                           [(c * 5 + k + j) % v for j, v in enumerate(sc.cross_feature_vocabs)],
                           [(c * 11 + 2 * k + j) % v for j, v in enumerate(sc.item_feature_vocabs)])
                 for c in range(1 + k % 5)]
        reqs.append(InferenceRequest(int(b["user_id"][u]), scenario, 1100 + 37 * k, hist, rt, cands))
    return reqs


def test_subgraph_registry_and_scoping():
    osch, ocfg, P = model("tiny_j")
    sch, cfg = from_oracle(osch, ocfg)
    m = Model(sch, cfg).restrict_to_scenario(1)
    names = [n for n, _, _ in m.param_specs()]
    assert names == [n for n in P if owner(n) in (-1, 1)]  # extract_subgraph keeps exactly these
    with pytest.raises(abi.ConfigError):
        m.set_param("head/s2/ctr/tower_b", np.zeros((1, 1), np.float32))
    with pytest.raises(abi.ConfigError):
        Model(sch, cfg).restrict_to_scenario(99)
    m.set_params({n: P[n] for n in names})
    reqs = _requests(batch("tiny_j"), sch, 2, 1)
    with pytest.raises(abi.IntegrityError):
        infer_request(m, reqs[0])


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_subgraph_requests_match_full_model_and_oracle(precision):
    osch, ocfg, P = model("tiny_j")
    sch, cfg = from_oracle(osch, ocfg)
    full = Model.build(sch, cfg, P, precision=precision)
    sub = Model.build_subgraph(sch, cfg, {n: v for n, v in P.items() if owner(n) in (-1, 1)}, 1,
                               precision=precision)
    reqs = _requests(batch("tiny_j"), sch, 1, 12)
    batched = infer_requests(sub, reqs)
    orc = O.Oracle(osch, ocfg, P, np.float64)
    for r, got in zip(reqs, batched):
        alone = infer_request(sub, r)
        via_full = infer_request(full, r)
        assert [(x.exposure_index, x.task) for x in got] == [(x.exposure_index, x.task) for x in alone]
        # batching and the subgraph restriction are bitwise neutral
        assert [x.probability for x in got] == [x.probability for x in alone]
        assert [x.probability for x in alone] == [x.probability for x in via_full]
        from paper_2602_11235_b200.schema import pack_samples, sample_view_of_request
        want = orc.forward_batch(pack_samples([sample_view_of_request(r)]))
        z = np.log(np.array([x.probability for x in got]) / (1 - np.array([x.probability for x in got])))
        zr = np.array([w[4] for w in want])
        assert [w[2] for w in want] == [x.exposure_index for x in got]
        tol = 1e-4 if precision == "fp32" else 8e-2  # bf16: storage error at O(1) logits (test_gpu_parity)
        assert np.max(np.abs(z - zr)) <= tol * max(1.0, float(np.max(np.abs(zr))))


def test_requests_batch_across_scenarios_on_full_model():
    osch, ocfg, P = model("tiny_j")
    sch, cfg = from_oracle(osch, ocfg)
    full = Model.build(sch, cfg, P)
    b = batch("tiny_j")
    reqs = _requests(b, sch, 0, 4) + _requests(b, sch, 1, 4) + _requests(b, sch, 3, 4)
    out = infer_requests(full, reqs)
    for r, got in zip(reqs, out):
        assert [x.probability for x in got] == [x.probability for x in infer_request(full, r)]
        assert all(x.scenario_id == r.scenario_id for x in got)
