"""Known-answer and size-independent properties of the CUDA path,
through the C ABI. Needs a B200.

Each test restates one of the reference's own known-answer tests on the GPU:
  zero-f2 identity          test_hta.cpp:268-286
  T isolation (full size)   test_hta.cpp:288-326, verify.hpp:440-481
  exposure permutation      test_tokenizer.cpp:194-219
  head isolation            test_heads_metrics.cpp:102-121
  uniform gate              test_heads_metrics.cpp:52-81
and, at the BASELINE small size (1024 users) where the numpy oracle is too
slow, the bf16 tensor-core path against the independent fp32 SIMT check path.
"""
import numpy as np
import pytest

import mtfm_oracle as O
from helpers import oracle_records, rel_err, to_oracle
from paper_2602_11235_b200 import Model, datagen
from paper_2602_11235_b200.schema import normalize_batch

pytestmark = pytest.mark.gpu


def _small(n_users, seed=5, precision="bf16", params=None):
    wl = datagen.WORKLOADS["small"]()
    b = datagen.generate(wl, n_users=n_users)
    m = Model(wl.schemas, wl.cfg, precision=precision)
    P = params if params is not None else datagen.random_params(m.param_specs(), seed=seed)
    m.set_params(P)
    return wl, b, m, P


def _append_exposure(b, u):
    """Batch with one extra exposure for user u: a copy of its first exposure,
    1 ms later (a distinct timestamp, so the canonical order is unambiguous)."""
    b = normalize_batch(b)
    x = int(b["exp_off"][u])
    f0, f1 = int(b["exp_feat_off"][x]), int(b["exp_feat_off"][x + 1])
    ins = int(b["exp_off"][u + 1])  # new exposure goes last in user u's list
    fins = int(b["exp_feat_off"][ins])
    out = dict(b)
    out["exp_off"] = b["exp_off"].copy()
    out["exp_off"][u + 1:] += 1
    out["exp_scenario"] = np.insert(b["exp_scenario"], ins, b["exp_scenario"][x])
    out["exp_ts"] = np.insert(b["exp_ts"], ins, int(b["exp_ts"].max()) + 1)
    blk = b["exp_blk"].reshape(-1, 3)
    out["exp_blk"] = np.insert(blk, ins, blk[x], axis=0).reshape(-1)
    out["exp_feats"] = np.insert(b["exp_feats"], fins, b["exp_feats"][f0:f1])
    fo = b["exp_feat_off"]
    out["exp_feat_off"] = np.concatenate([fo[:ins + 1], fo[ins:] + (f1 - f0)])
    return normalize_batch(out)


def test_zero_f2_identity():
    """f2_w = f2_b = 0 makes every HTA layer the identity on X (test_hta.cpp:268-286):
    the final X equals the tokenizer output X0 of the oracle, row for row."""
    wl = datagen.WORKLOADS["small"]()
    b = datagen.generate(wl, n_users=3)
    m = Model(wl.schemas, wl.cfg, precision="fp32")
    P = datagen.random_params(m.param_specs(), seed=9)
    for k in P:
        if k.endswith("/f2_w") or k.endswith("/f2_b"):
            P[k] = np.zeros_like(P[k])
    m.set_params(P)
    pb = m.prepare(b)
    pb.run()
    pb.results()
    n_ev, n_x = len(b["ev_ts"]), len(b["exp_ts"])
    d = wl.cfg.hta.d_model
    X = pb.fetch("x", np.float32, (n_ev + n_x) * d).reshape(-1, d)
    osch, ocfg = to_oracle(wl.schemas, wl.cfg)
    orc = O.Oracle(osch, ocfg, P, np.float64)
    for u, v in enumerate(O.user_views(b)):
        r = orc.forward_user(v)
        lh, lr, lt = r["plan"].bounds
        ev0, x0 = b["ev_off"][b["seq_off"][u]], b["exp_off"][u]
        got = np.concatenate([X[ev0:ev0 + lh + lr], X[n_ev + x0:n_ev + x0 + lt]])
        assert np.allclose(r["xf"], r["x0"])  # the oracle agrees that the stack is the identity
        assert np.max(np.abs(got - r["x0"])) <= 1e-4 * max(1.0, np.max(np.abs(r["x0"])))


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_t_isolation_full_size(precision):
    """Adding a T token to one user changes no other record (T rows never see each
    other; test_hta.cpp:288-326): bitwise, at the BASELINE small size."""
    n_users = 1024 if precision == "bf16" else 96
    wl, b, m, P = _small(n_users, precision=precision)
    base = m.forward_batch(b)
    u = 7
    ext = m.forward_batch(_append_exposure(b, u))
    n_new = len(ext.logit) - len(base.logit)
    assert n_new == len(wl.schemas.scenarios[int(b["exp_scenario"][b["exp_off"][u]])].tasks)
    # every original record is present with the identical logit
    key = lambda r: list(zip(r.user_id.tolist(), r.scenario_id.tolist(), r.exposure_index.tolist(),
                             r.task_index.tolist()))
    pos = {k: i for i, k in enumerate(key(ext))}
    idx = np.array([pos[k] for k in key(base)])
    assert np.array_equal(ext.logit[idx], base.logit)
    assert np.array_equal(ext.probability[idx], base.probability)


def test_exposure_permutation_invariance():
    """Listing a user's exposures in another order changes nothing but the
    exposure indices (canonical T order, test_tokenizer.cpp:194-219)."""
    wl, b, m, P = _small(64)
    b = normalize_batch(b)
    rng = np.random.default_rng(3)
    # distinct timestamps so the canonical (ts, scenario, index) order has no ties
    b["exp_ts"] = b["exp_ts"] * 4096 + np.arange(len(b["exp_ts"])) % 4096
    base = m.forward_batch(b)
    perm_b = {k: v.copy() for k, v in b.items()}
    new_of_old = np.arange(len(b["exp_ts"]))
    blk = b["exp_blk"].reshape(-1, 3)
    feats, fo = [], [0]
    order_all = []
    for u in range(len(b["user_id"])):
        x0, x1 = b["exp_off"][u], b["exp_off"][u + 1]
        order = x0 + rng.permutation(x1 - x0)
        order_all.extend(order.tolist())
        new_of_old[order] = np.arange(x0, x1)
    order_all = np.array(order_all, np.int64)
    perm_b["exp_scenario"] = b["exp_scenario"][order_all]
    perm_b["exp_ts"] = b["exp_ts"][order_all]
    perm_b["exp_blk"] = blk[order_all].reshape(-1)
    for x in order_all:
        seg = b["exp_feats"][b["exp_feat_off"][x]:b["exp_feat_off"][x + 1]]
        feats.append(seg)
        fo.append(fo[-1] + len(seg))
    perm_b["exp_feats"] = np.concatenate(feats).astype(b["exp_feats"].dtype)
    perm_b["exp_feat_off"] = np.array(fo, dtype=b["exp_feat_off"].dtype)
    got = m.forward_batch(normalize_batch(perm_b))
    # same records in the same (canonical) order; exposure indices follow the permutation
    assert np.array_equal(got.user_id, base.user_id)
    assert np.array_equal(got.scenario_id, base.scenario_id)
    assert np.array_equal(got.task_index, base.task_index)
    u_of = {int(uid): u for u, uid in enumerate(b["user_id"])}
    off = np.array([b["exp_off"][u_of[int(uid)]] for uid in base.user_id], np.int64)
    assert np.array_equal(got.exposure_index, new_of_old[base.exposure_index + off] - off)
    assert np.array_equal(got.logit, base.logit)


def test_head_isolation():
    """Changing one scenario's head weights changes only that scenario's records
    (test_heads_metrics.cpp:102-121)."""
    wl, b, m, P = _small(32)
    base = m.forward_batch(b)
    sid = wl.schemas.scenarios[1].scenario_id
    P2 = dict(P)
    for k in P:
        if k.startswith(f"head/s{sid}/"):
            P2[k] = P[k] * 1.5 + 0.1
    m.set_params(P2)
    got = m.forward_batch(b)
    other = base.scenario_id != sid
    assert np.array_equal(got.logit[other], base.logit[other])
    assert np.max(np.abs(got.logit[~other] - base.logit[~other])) > 1e-3


def test_uniform_gate():
    """Zero gate weights and biases give every expert weight 1/E
    (test_heads_metrics.cpp:52-81): fp32 check mode against the oracle."""
    wl = datagen.WORKLOADS["small"]()
    b = datagen.generate(wl, n_users=4)
    m = Model(wl.schemas, wl.cfg, precision="fp32")
    P = datagen.random_params(m.param_specs(), seed=11)
    for k in P:
        if k.endswith("/gate_w") or k.endswith("/gate_b"):
            P[k] = np.zeros_like(P[k])
    m.set_params(P)
    osch, ocfg = to_oracle(wl.schemas, wl.cfg)
    keys, z_ref, _ = oracle_records(osch, ocfg, P, b)
    ra = m.forward_batch(b)
    assert rel_err(ra.logit.astype(np.float64), z_ref) <= 1e-4


def test_bf16_vs_fp32_check_full_size():
    """At the BASELINE small size the bf16 tensor-core path and the independent
    fp32 SIMT check path agree within the bf16 logit tolerance."""
    wl = datagen.WORKLOADS["small"]()
    b = datagen.generate(wl, n_users=1024)
    m16 = Model(wl.schemas, wl.cfg, precision="bf16")
    P = datagen.random_params(m16.param_specs(), seed=5)
    m16.set_params(P)
    m32 = Model.build(wl.schemas, wl.cfg, P, precision="fp32")
    a16 = m16.forward_batch(b)
    a32 = m32.forward_batch(b)
    assert np.array_equal(a16.user_id, a32.user_id) and np.array_equal(a16.exposure_index, a32.exposure_index)
    assert np.max(np.abs(a16.logit - a32.logit)) <= 2e-2
