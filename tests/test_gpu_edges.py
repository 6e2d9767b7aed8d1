"""Edge cases of the CUDA path (through the C ABI): ragged and empty users,
empty batches, the scenario-scoped forward, long users and users above the
planning CTA's SMEM capacity. Needs a B200. Expected values come from the pinned numpy oracle or
from the reference's own rules (tokenizer.hpp:240-268 for empty samples,
model.hpp:244-312 for the scoped forward)."""
import dataclasses

import numpy as np
import pytest

from helpers import oracle_records, rel_err, to_oracle
from paper_2602_11235_b200 import Model, abi, datagen
from paper_2602_11235_b200.schema import normalize_batch, param_specs
from paper_2602_11235_b200.shard import take_users

pytestmark = pytest.mark.gpu


def _wl(name="small", **kw):
    return dataclasses.replace(datagen.WORKLOADS[name](), **kw)


def _model(wl, precision="bf16", seed=5):
    m = Model(wl.schemas, wl.cfg, precision=precision)
    P = datagen.random_params(m.param_specs(), seed=seed)
    m.set_params(P)
    return m, P


def _cat(*batches):
    """Concatenate packed batches user-wise (include/mtfm_cuda.h layout)."""
    bs = [normalize_batch(b) for b in batches]
    out = {}
    for k in ("user_id", "seq_kind", "seq_schema", "ev_ts", "ev_feats", "exp_scenario", "exp_ts", "exp_blk",
              "exp_feats"):
        out[k] = np.concatenate([b[k] for b in bs])
    out["user_id"] = np.arange(len(out["user_id"]), dtype=np.int64)

    def offs(key, counts_key=None):
        parts, base = [np.zeros(1, np.int64)], 0
        for b in bs:
            o = b[key].astype(np.int64)
            parts.append(o[1:] + base)
            base += int(o[-1])
        return np.concatenate(parts)
    for k in ("seq_off", "ev_off", "ev_feat_off", "exp_off", "exp_feat_off"):
        out[k] = offs(k)
    return normalize_batch(out)


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_ragged_users_vs_oracle(precision):
    """Users without events (targets attend only to themselves), users without
    exposures (no records) and ordinary users in one batch."""
    wl = _wl()
    no_ev = datagen.generate(_wl(hist_len=0, rt_len=0, exp_per_scen=2, seed=21), n_users=2)
    no_x = datagen.generate(_wl(hist_len=40, rt_len=9, exp_per_scen=0, seed=22), n_users=2)
    ragged = datagen.generate(_wl(hist_len=("lognormal", 30, 1.0, 1, 300), rt_len=("lognormal", 8, 1.0, 0, 64),
                                  exp_per_scen=("lognormal", 5, 0.8, 1, 20), seed=23), n_users=4)
    b = _cat(no_ev, ragged, no_x)
    m, P = _model(wl, precision)
    osch, ocfg = to_oracle(wl.schemas, wl.cfg)
    keys, z_ref, _ = oracle_records(osch, ocfg, P, b)
    ra = m.forward_batch(b)
    assert np.array_equal(np.stack([ra.user_id, ra.scenario_id, ra.exposure_index, ra.task_index], 1), keys)
    if precision == "bf16":
        assert np.max(np.abs(ra.logit - z_ref)) <= 2e-2
    else:
        assert rel_err(ra.logit.astype(np.float64), z_ref) <= 1e-4


def test_empty_batch_and_sample_without_tokens():
    wl = _wl()
    m, _ = _model(wl)
    b = datagen.generate(wl, n_users=3)
    empty = take_users(b, np.zeros(0, np.int64))
    assert len(m.forward_batch(empty).logit) == 0
    # a user with neither events nor exposures: contract_error (tokenizer.hpp:240-268)
    none = datagen.generate(_wl(hist_len=0, rt_len=0, exp_per_scen=0, seed=3), n_users=1)
    with pytest.raises(abi.ContractError):
        m.forward_batch(_cat(b, none))


def test_scoped_forward():
    """forward_scoped(only_scenario) (model.hpp:284-311): a sample whose exposures
    all belong to the scenario scores exactly as unscoped; another scenario in
    the sample is an integrity_error (the scenario subgraph has no tokenizer for it)."""
    wl = _wl()
    m, _ = _model(wl)
    b = normalize_batch(datagen.generate(wl, n_users=8))
    sid = int(wl.schemas.scenarios[2].scenario_id)
    keep = np.nonzero(b["exp_scenario"] == sid)[0]
    # batch restricted to one scenario's exposures
    one = dict(b)
    cnt = np.array([np.sum((keep >= b["exp_off"][u]) & (keep < b["exp_off"][u + 1]))
                    for u in range(len(b["user_id"]))])
    one["exp_off"] = np.concatenate([[0], np.cumsum(cnt)])
    one["exp_scenario"] = b["exp_scenario"][keep]
    one["exp_ts"] = b["exp_ts"][keep]
    one["exp_blk"] = b["exp_blk"].reshape(-1, 3)[keep].reshape(-1)
    fo = b["exp_feat_off"]
    one["exp_feats"] = np.concatenate([b["exp_feats"][fo[x]:fo[x + 1]] for x in keep])
    one["exp_feat_off"] = np.concatenate([[0], np.cumsum([fo[x + 1] - fo[x] for x in keep])])
    one = normalize_batch(one)
    full = m.forward_batch(one)
    scoped = m.forward_batch(one, only_scenario=sid)
    assert np.array_equal(scoped.logit, full.logit)
    assert (scoped.scenario_id == sid).all()
    with pytest.raises(abi.IntegrityError):
        m.forward_batch(b, only_scenario=sid)


def test_long_user_vs_oracle():
    """One user far beyond the small shape (2 x 1500 history + 600 realtime +
    100 targets): attention spans many key tiles and query tiles."""
    wl = _wl(hist_len=1500, rt_len=600, exp_per_scen=25, seed=31)
    b = datagen.generate(wl, n_users=1)
    m, P = _model(wl)
    osch, ocfg = to_oracle(wl.schemas, wl.cfg)
    keys, z_ref, _ = oracle_records(osch, ocfg, P, b)
    ra = m.forward_batch(b)
    assert np.array_equal(np.stack([ra.user_id, ra.scenario_id, ra.exposure_index, ra.task_index], 1), keys)
    assert np.max(np.abs(ra.logit - z_ref)) <= 2e-2


@pytest.fixture(scope="module")
def above_capacity_case():
    long_u = datagen.generate(_wl("tiny", hist_len=6000, rt_len=1000, exp_per_scen=3, seed=41), n_users=1)
    short = datagen.generate(_wl("tiny", seed=42), n_users=3)
    b = _cat(short, long_u)
    wl = _wl("tiny")
    P = datagen.random_params(param_specs(wl.schemas, wl.cfg), seed=5)
    osch, ocfg = to_oracle(wl.schemas, wl.cfg)
    keys, z_ref, _ = oracle_records(osch, ocfg, P, b)  # ~40 s of numpy (13 000^2 masks)
    return wl, P, b, keys, z_ref


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_user_above_plan_smem_capacity_vs_oracle(precision, above_capacity_case):
    """A user with 13 000 context tokens (more than the 12 288 a planning CTA sorts
    in SMEM) is planned from a global scratch slice, next to ordinary users planned
    in SMEM in the same launch; records match the oracle."""
    wl, P, b, keys, z_ref = above_capacity_case
    m = Model(wl.schemas, wl.cfg, precision=precision)
    m.set_params(P)
    ra = m.forward_batch(b)
    assert np.array_equal(np.stack([ra.user_id, ra.scenario_id, ra.exposure_index, ra.task_index], 1), keys)
    if precision == "fp32":
        assert rel_err(ra.logit, z_ref) <= 1e-4
    else:
        assert np.max(np.abs(ra.logit - z_ref)) <= 2e-2


def test_context_timestamp_below_minus_one_is_dimension_error():
    """check_meta_order (token_types.hpp:53-72): within the H and R blocks time must not
    fall below the block's starting value -1, so an event at t = -5 makes plan_tokens
    throw dimension_error before any tokenizer check; t = -1 is accepted."""
    from golden_util import batch, model
    from helpers import from_oracle
    from paper_2602_11235_b200 import Model, abi
    osch, ocfg, P = model("tiny")
    sch, cfg = from_oracle(osch, ocfg)
    m = Model.build(sch, cfg, P, precision="fp32")
    b = {k: v.copy() for k, v in batch("tiny").items()}
    u = 2
    e0 = b["ev_off"][b["seq_off"][u]]
    b["ev_ts"][e0] = -1
    m.forward_batch(b)  # -1 is fine
    b["ev_ts"][e0] = -5
    b["exp_feats"][b["exp_feat_off"][b["exp_off"][u]]] = 10 ** 6  # a later lookup error of the same user
    with pytest.raises(abi.DimensionError) as ei:
        m.forward_batch(b)
    assert "user index 2" in str(ei.value) and "time-sorted" in str(ei.value)


def _permute_sequence(b, seq, order):
    """Reorder the events of packed sequence `seq` (timestamps with their features)."""
    b = {k: v.copy() for k, v in b.items()}
    e0, e1 = int(b["ev_off"][seq]), int(b["ev_off"][seq + 1])
    fo = b["ev_feat_off"]
    feats = [b["ev_feats"][fo[e]:fo[e + 1]] for e in range(e0, e1)]
    ts = b["ev_ts"][e0:e1].copy()
    new_feats = [feats[i] for i in order]
    b["ev_ts"][e0:e1] = ts[order]
    pos = int(fo[e0])
    for k, f in enumerate(new_feats):
        b["ev_feats"][pos:pos + len(f)] = f
        pos += len(f)
        b["ev_feat_off"][e0 + k + 1] = pos
    return normalize_batch(b)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_unsorted_sequences_and_cross_sequence_ties_vs_oracle(precision):
    """plan_tokens stable-sorts each kind's context events by time (tokenizer.hpp:117-123):
    sequences in time order take the merge path of the plan kernel, a shuffled sequence
    the bitonic sort; equal timestamps across the two H sequences keep pile order."""
    wl = _wl(hist_len=60, rt_len=12, exp_per_scen=3, seed=51)
    b = datagen.generate(wl, n_users=4)
    # user 1: shuffle its first sequence; user 2: copy timestamps of its first H sequence
    # into its second so that every event ties with one of the other sequence
    s1 = int(b["seq_off"][1])
    n1 = int(b["ev_off"][s1 + 1] - b["ev_off"][s1])
    b = _permute_sequence(b, s1, np.random.default_rng(5).permutation(n1))
    s2 = int(b["seq_off"][2])
    a0, a1 = int(b["ev_off"][s2]), int(b["ev_off"][s2 + 1])
    c0, c1 = int(b["ev_off"][s2 + 1]), int(b["ev_off"][s2 + 2])
    k = min(a1 - a0, c1 - c0)
    ts = np.sort(b["ev_ts"][a0:a0 + k])
    b["ev_ts"][a0:a0 + k] = ts
    b["ev_ts"][c0:c0 + k] = ts
    b["ev_ts"][a0 + k:a1] = np.maximum(b["ev_ts"][a0 + k:a1], ts[-1])
    b["ev_ts"][c0 + k:c1] = np.maximum(b["ev_ts"][c0 + k:c1], ts[-1])
    assert b["seq_kind"][s2] == 0 and b["seq_kind"][s2 + 1] == 0
    m, P = _model(wl, precision)
    osch, ocfg = to_oracle(wl.schemas, wl.cfg)
    keys, z_ref, _ = oracle_records(osch, ocfg, P, b)
    ra = m.forward_batch(b)
    assert np.array_equal(np.stack([ra.user_id, ra.scenario_id, ra.exposure_index, ra.task_index], 1), keys)
    if precision == "bf16":
        assert np.max(np.abs(ra.logit - z_ref)) <= 2e-2
    else:
        assert rel_err(ra.logit.astype(np.float64), z_ref) <= 1e-4
