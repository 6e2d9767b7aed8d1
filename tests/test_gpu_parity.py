"""Parity of the CUDA path (through the C ABI) against the reference goldens
and the pinned numpy oracle. Needs a B200.

Tolerances (BASELINE.json north_star):
  fp32 check mode : max |z - z_ref| / max(|z_ref|, floor) <= 1e-4 on logits
                    (floor: helpers.check_floor, 1e-2 default-init / 1.0 jittered)
  bf16 fast mode  : default-init fixtures (|z| < 0.15): max |z - z_ref| <= 2e-2.
                    Jittered fixtures (O(1) logits): bf16 *storage* alone moves the
                    logits by up to ~0.12 (oracle/bf16_emu.py rounds at exactly the
                    fast path's storage points, in exact arithmetic otherwise). The
                    GPU's hardware SiLU (tanh.approx, ~2^-11 relative) re-rounds a
                    share of the bf16 values differently, so GPU and emulation are
                    two draws of the same storage noise, not bit-twins: the GPU is
                    held to the emulation's error statistics against the reference,
                    max |z - z_ref| <= 2 max |z_emu - z_ref| + 2e-2 and
                    rms(z - z_ref) <= 1.5 rms(z_emu - z_ref) + 1e-3.
  integer plan    : bit-exact
The *_j fixtures carry parameters moved off the reference's default init
(every bias, GLN gain/bias, O(1) logits; oracle/ref_dump.cpp --jitter).
Observed errors are printed (run with -rA to see them in the log).
"""
import numpy as np
import pytest

import mtfm_oracle as O
from golden_util import JITTERED, NAMES, batch, load, model, ref_records
from helpers import check_floor, from_oracle, oracle_records, rel_err, to_oracle
from paper_2602_11235_b200 import Model, abi, datagen

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-4
BF16_TOL = 2e-2
ALL = NAMES + JITTERED
BF16_OK = [n for n in ALL if n != "micro"]  # micro has head_dim 8 (< 16): fp32 check mode only


def _build(name, precision):
    osch, ocfg, P = model(name)
    sch, cfg = from_oracle(osch, ocfg)
    return Model.build(sch, cfg, P, precision=precision)


@pytest.mark.parametrize("name", ALL)
def test_golden_fp32_check_mode(name):
    m = _build(name, "fp32")
    ra = m.forward_batch(batch(name))
    keys, z64, z32, p64, p32 = ref_records(name)
    got = np.stack([ra.user_id, ra.scenario_id, ra.exposure_index, ra.task_index], 1)
    assert np.array_equal(got, keys)
    fl = check_floor(name)
    err = rel_err(ra.logit.astype(np.float64), z64, fl)
    ref_err = rel_err(z32, z64, fl)
    dp = float(np.max(np.abs(ra.probability - p64)))
    print(f"fp32 {name}: rel err {err:.3e} (floor {fl}; reference Model<float>: {ref_err:.3e}), "
          f"max |dz| {np.max(np.abs(ra.logit - z64)):.3e}, max |dp| {dp:.3e}, max |z| {np.max(np.abs(z64)):.2f}")
    assert err <= FP32_TOL
    assert dp <= 1e-5


@pytest.mark.parametrize("name", BF16_OK)
def test_golden_bf16(name):
    m = _build(name, "bf16")
    ra = m.forward_batch(batch(name))
    keys, z64, *_ = ref_records(name)
    got = np.stack([ra.user_id, ra.scenario_id, ra.exposure_index, ra.task_index], 1)
    assert np.array_equal(got, keys)
    z = ra.logit.astype(np.float64)
    dz = float(np.max(np.abs(z - z64)))
    import bf16_emu
    osch, ocfg, P = model(name)
    z_emu = np.array([r[4] for r in bf16_emu.Bf16Oracle(osch, ocfg, P).forward_batch(batch(name))])
    d_emu = float(np.max(np.abs(z - z_emu)))
    d_store = float(np.max(np.abs(z_emu - z64)))
    rms = float(np.sqrt(np.mean((z - z64) ** 2)))
    rms_store = float(np.sqrt(np.mean((z_emu - z64) ** 2)))
    print(f"bf16 {name}: max |z - z_ref| {dz:.3e} (rms {rms:.3e}); bf16 storage alone (emulation) max "
          f"{d_store:.3e} (rms {rms_store:.3e}); max |z - z_emu| {d_emu:.3e}; max |z| {np.max(np.abs(z64)):.2f}")
    if name.endswith("_j"):
        assert dz <= 2 * d_store + BF16_TOL
        assert rms <= 1.5 * rms_store + 1e-3
    else:
        assert dz <= BF16_TOL


@pytest.mark.parametrize("name", ALL)
@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_plan_bit_exact(name, precision):
    if precision == "bf16" and name not in BF16_OK:
        pytest.skip("head_dim < 16")
    a = load(name)
    m = _build(name, precision)
    b = batch(name)
    pb = m.prepare(b)
    pb.run()
    pb.results()
    n_ev, n_x = len(b["ev_ts"]), len(b["exp_ts"])
    R = n_ev + n_x
    item = pb.fetch("item", np.int32, R)
    prefix = pb.fetch("prefix", np.int32, R)
    self_ = pb.fetch("self", np.int32, R)
    src = pb.fetch("src", np.int32, R)
    scale = pb.fetch("scale", np.float32, R)
    for u in range(len(b["user_id"])):
        o0, o1 = a["plan/off"][u], a["plan/off"][u + 1]
        lh, lr, lt = a["plan/bounds"][u]
        ev0 = b["ev_off"][b["seq_off"][u]]
        x0 = b["exp_off"][u]
        f2p = a["plan/final_to_pile"][o0:o1]
        vc = a["plan/valid_count"][o0:o1]
        tg = a["plan/token_group"][o0:o1]
        ctx = slice(ev0, ev0 + lh + lr)
        tr = slice(n_ev + x0, n_ev + x0 + lt)
        # context rows: final order -> pile row == local event index
        assert np.array_equal(item[ctx], ev0 + f2p[:lh + lr])
        assert np.array_equal(prefix[ctx], vc[:lh + lr])
        assert np.array_equal(src[ctx], tg[:lh + lr])
        assert (self_[ctx] == -1).all()
        # T rows: canonical order, exposure_ref
        assert np.array_equal(item[tr], x0 + a["plan/exposure_ref"][o0 + lh + lr:o1])
        assert np.array_equal(prefix[tr] + 1, vc[lh + lr:])
        assert np.array_equal(src[tr], tg[lh + lr:])
        assert np.array_equal(self_[tr], np.arange(tr.start, tr.stop))
        # row scale (hta.hpp:53-67), float32 exact
        osch, ocfg, _ = model(name)
        if ocfg.norm == "valid":
            want = (np.float32(1) / np.maximum(vc, 1).astype(np.float32)).astype(np.float32)
        elif ocfg.norm == "seqlen":
            want = np.full(len(vc), np.float32(1) / np.float32(len(vc)), np.float32)
        else:
            want = np.ones(len(vc), np.float32)
        got = np.concatenate([scale[ctx], scale[tr]])
        assert np.array_equal(got, want)


@pytest.mark.parametrize("name,n_users", [("small", 6), ("base", 6), ("large", 2), ("paper", 2)])
def test_synthetic_configs_vs_oracle(name, n_users):
    wl = datagen.WORKLOADS[name]()
    b = datagen.generate(wl, n_users=n_users)
    osch, ocfg = to_oracle(wl.schemas, wl.cfg)
    m16 = Model(wl.schemas, wl.cfg, precision="bf16")
    P = datagen.random_params(m16.param_specs(), seed=5)
    m16.set_params(P)
    keys, z_ref, _ = oracle_records(osch, ocfg, P, b)
    ra = m16.forward_batch(b)
    assert np.array_equal(np.stack([ra.user_id, ra.scenario_id, ra.exposure_index, ra.task_index], 1), keys)
    e16 = float(np.max(np.abs(ra.logit - z_ref)))
    m32 = Model.build(wl.schemas, wl.cfg, P, precision="fp32")
    rb = m32.forward_batch(b)
    e32 = rel_err(rb.logit.astype(np.float64), z_ref)
    print(f"synthetic {name}: bf16 max |dz| {e16:.3e}, fp32 rel err {e32:.3e}, max |z| {np.max(np.abs(z_ref)):.3f}")
    assert e16 <= BF16_TOL
    assert e32 <= FP32_TOL


def test_error_taxonomy_and_order():
    m = _build("tiny", "bf16")
    b = {k: v.copy() for k, v in batch("tiny").items()}
    # out-of-vocab id in user 3's first event -> lookup_error (eval_ctx.hpp:193-194)
    e = b["ev_off"][b["seq_off"][3]]
    b["ev_feats"][b["ev_feat_off"][e]] = 10 ** 6
    with pytest.raises(abi.LookupError_) as ei:
        m.forward_batch(b)
    assert "user index 3" in str(ei.value)
    # unknown scenario in user 1 -> integrity_error (tokenizer.hpp:255-258); user 1 is reported first
    x = b["exp_off"][1]
    b["exp_scenario"][x] = 99
    with pytest.raises(abi.IntegrityError) as ei:
        m.forward_batch(b)
    assert "user index 1" in str(ei.value)


def test_missing_slot_is_dimension_error():
    m = _build("tiny", "fp32")
    b = {k: v.copy() for k, v in batch("tiny").items()}
    x = b["exp_off"][2]
    b["exp_blk"][3 * x] = 0  # drop the user-feature block of one exposure
    with pytest.raises(abi.DimensionError):
        m.forward_batch(b)


def test_unknown_parameter_and_shape():
    osch, ocfg, P = model("tiny")
    sch, cfg = from_oracle(osch, ocfg)
    m = Model(sch, cfg)
    with pytest.raises(abi.ConfigError):
        m.set_param("hta/b9/l0/f1_w", np.zeros((64, 64), np.float32))
    with pytest.raises(abi.DimensionError):
        m.set_param("hta/b0/l1/f1_w", np.zeros((3, 3), np.float32))


def test_aggregation_equivalence():
    """T tokens never see each other, so aggregated scoring equals singleton
    scoring (verify.hpp:440-481), here through the bf16 kernels."""
    from paper_2602_11235_b200.schema import normalize_batch
    m = _build("tiny", "bf16")
    b = batch("tiny")
    agg = m.forward_batch(b)
    for u in range(len(b["user_id"])):
        x0, x1 = b["exp_off"][u], b["exp_off"][u + 1]
        s0, s1 = b["seq_off"][u], b["seq_off"][u + 1]
        e0, e1 = b["ev_off"][s0], b["ev_off"][s1]
        for x in range(x0, x1):
            single = dict(
                user_id=b["user_id"][u:u + 1], seq_off=np.array([0, s1 - s0]), seq_kind=b["seq_kind"][s0:s1],
                seq_schema=b["seq_schema"][s0:s1], ev_off=b["ev_off"][s0:s1 + 1] - e0, ev_ts=b["ev_ts"][e0:e1],
                ev_feat_off=b["ev_feat_off"][e0:e1 + 1] - b["ev_feat_off"][e0],
                ev_feats=b["ev_feats"][b["ev_feat_off"][e0]:b["ev_feat_off"][e1]],
                exp_off=np.array([0, 1]), exp_scenario=b["exp_scenario"][x:x + 1], exp_ts=b["exp_ts"][x:x + 1],
                exp_feat_off=b["exp_feat_off"][x:x + 2] - b["exp_feat_off"][x], exp_blk=b["exp_blk"][3 * x:3 * x + 3],
                exp_feats=b["exp_feats"][b["exp_feat_off"][x]:b["exp_feat_off"][x + 1]])
            solo = m.forward_batch(normalize_batch(single))
            sel = (agg.user_id == b["user_id"][u]) & (agg.exposure_index == x - x0)
            assert np.max(np.abs(agg.logit[sel] - solo.logit)) <= 2e-3
