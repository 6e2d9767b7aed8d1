"""aggregate_users (datagen.cpp:171-216): the exposure stream grouped per user
(scenario ascending, stream order within), users ascending, joined with the
shared H/R store — bit-exact against the reference's own outputs
(tests/golden/agg.npz, oracle/ref_agg.cpp), including its integrity errors.
CPU: the numpy restatement. GPU: mtfm_cuda_aggregate_users through the C ABI."""
import numpy as np
import pytest

import mtfm_oracle as O
from golden_util import GOLDEN
from paper_2602_11235_b200.schema import BATCH_KEYS

STREAM_KEYS = ("user_id", "scenario", "ts", "feat_off", "blk", "feats")


def _cases():
    a = np.load(f"{GOLDEN}/agg.npz")
    g = {k.replace("__", "/"): a[k] for k in a.files}
    out = []
    for k in range(int(g["n_cases"][0])):
        p = f"c{k}/"
        out.append(dict(
            scen_ids=g[p + "scen_ids"],
            stream={s: g[p + "stream/" + s] for s in STREAM_KEYS},
            store={s: g[p + "store/" + s] for s in BATCH_KEYS},
            error=bytes(g[p + "error"]).decode(),
            out={s: g[p + "out/" + s] for s in BATCH_KEYS} if not bytes(g[p + "error"]) else None,
            report=g.get(p + "report")))
    return out


CASES = _cases()


def _same(got, want):
    for k in BATCH_KEYS:
        assert np.array_equal(np.asarray(got[k], np.int64), np.asarray(want[k], np.int64)), k


@pytest.mark.parametrize("k", range(len(CASES)))
def test_oracle_aggregate_matches_reference(k):
    c = CASES[k]
    if c["error"]:
        with pytest.raises(O.IntegrityError) as ei:
            O.aggregate_users(c["scen_ids"], c["stream"], c["store"])
        assert str(ei.value) == c["error"]
        return
    out, src = O.aggregate_users(c["scen_ids"], c["stream"], c["store"])
    _same(out, c["out"])
    assert len(src) == int(c["report"][0])


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(len(CASES)))
def test_gpu_aggregate_bit_exact(k):
    from paper_2602_11235_b200 import abi, aggregate_users
    c = CASES[k]
    if c["error"]:
        with pytest.raises(abi.IntegrityError) as ei:
            aggregate_users(c["scen_ids"], c["stream"], c["store"])
        assert str(ei.value) == c["error"]
        return
    out, src, rep = aggregate_users(c["scen_ids"], c["stream"], c["store"])
    _same(out, c["out"])
    assert rep["n_exposure_records"] == int(c["report"][0]) and rep["n_user_samples"] == int(c["report"][1])
    # exp_src: every output exposure is its stream element (labels are joined through it)
    _, want_src = O.aggregate_users(c["scen_ids"], c["stream"], c["store"])
    assert np.array_equal(src, np.asarray(want_src, np.int32))


@pytest.mark.gpu
def test_gpu_aggregate_store_order_is_checked():
    from paper_2602_11235_b200 import abi, aggregate_users
    c = CASES[2]
    store = {k: v.copy() for k, v in c["store"].items()}
    store["user_id"] = store["user_id"][::-1].copy()
    with pytest.raises(abi.ContractError):
        aggregate_users(c["scen_ids"], c["stream"], store)


@pytest.mark.gpu
def test_gpu_aggregate_at_scale_feeds_the_forward():
    """1024 users x 32 exposures streamed in a shuffled order -> the GPU
    aggregation equals the restatement and scores like the direct batch."""
    from paper_2602_11235_b200 import Model, aggregate_users, datagen
    from paper_2602_11235_b200.schema import normalize_batch
    wl = datagen.WORKLOADS["small"]()
    b = datagen.generate(wl, n_users=1024)
    rng = np.random.default_rng(3)
    n = len(b["exp_ts"])
    user_of = np.repeat(b["user_id"], np.diff(b["exp_off"]))
    order = rng.permutation(n)
    foff = b["exp_feat_off"]
    stream = dict(user_id=user_of[order], scenario=b["exp_scenario"][order], ts=b["exp_ts"][order],
                  blk=b["exp_blk"].reshape(-1, 3)[order].reshape(-1))
    lens = (foff[1:] - foff[:-1])[order]
    stream["feat_off"] = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    stream["feats"] = np.concatenate([b["exp_feats"][foff[x]:foff[x + 1]] for x in order]).astype(np.int32)
    store = {k: b[k] for k in BATCH_KEYS}
    store.update(exp_off=np.zeros(len(b["user_id"]) + 1, np.int32), exp_scenario=np.zeros(0, np.int32),
                 exp_ts=np.zeros(0, np.int64), exp_feat_off=np.zeros(1, np.int32), exp_blk=np.zeros(0, np.int32),
                 exp_feats=np.zeros(0, np.int32))
    scen = [s.scenario_id for s in wl.schemas.scenarios]
    out, src, rep = aggregate_users(scen, stream, store)
    want, _ = O.aggregate_users(scen, stream, normalize_batch(store))
    _same(out, want)
    assert rep["n_user_samples"] == 1024 and rep["compression_ratio"] == pytest.approx(32.0)
    m = Model(wl.schemas, wl.cfg, precision="bf16")
    m.set_params(datagen.random_params(m.param_specs(), seed=7))
    ra = m.forward_batch(out)
    assert len(ra) == m.forward_batch(b).__len__()
