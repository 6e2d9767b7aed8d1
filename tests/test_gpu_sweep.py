"""The SURVEY §8(d) sweep axes on the CUDA path, against the pinned numpy
oracle: layer mixes (K:P) in {(0:1), (1:1), (3:1), (5:1), (3:0)} (bench.hpp:43-58),
targets per user in {4, 16, 64, 256} and the three AttnNorm row scales
(model_config.hpp:18-24). Small users so the oracle finishes in seconds; the
model width is the BASELINE small one (d=256, H=8, G=2). Needs a B200."""
import dataclasses

import numpy as np
import pytest

from helpers import oracle_records, rel_err, to_oracle
from paper_2602_11235_b200 import Model, datagen

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2
FP32_TOL = 1e-4


def _run(wl, n_users, precision):
    b = datagen.generate(wl, n_users=n_users)
    m = Model(wl.schemas, wl.cfg, precision=precision)
    P = datagen.random_params(m.param_specs(), seed=13)
    m.set_params(P)
    osch, ocfg = to_oracle(wl.schemas, wl.cfg)
    keys, z_ref, _ = oracle_records(osch, ocfg, P, b)
    ra = m.forward_batch(b)
    assert np.array_equal(np.stack([ra.user_id, ra.scenario_id, ra.exposure_index, ra.task_index], 1), keys)
    if precision == "bf16":
        assert np.max(np.abs(ra.logit - z_ref)) <= BF16_TOL
    else:
        assert rel_err(ra.logit.astype(np.float64), z_ref) <= FP32_TOL


def _wl(K, P, blocks=1, norm="valid", **kw):
    wl = datagen.WORKLOADS["small"]()
    hta = dataclasses.replace(wl.cfg.hta, target_layers=K, full_layers=P, blocks=blocks, norm=norm)
    kw.setdefault("hist_len", 60)
    kw.setdefault("rt_len", 20)
    kw.setdefault("exp_per_scen", 3)
    return dataclasses.replace(wl, cfg=dataclasses.replace(wl.cfg, hta=hta), **kw)


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
@pytest.mark.parametrize("K,P,blocks", [(0, 1, 2), (1, 1, 1), (3, 1, 2), (5, 1, 1), (3, 0, 1), (3, 0, 2), (2, 0, 3), (1, 2, 2), (0, 3, 1), (2, 2, 1)])
def test_layer_mix(K, P, blocks, precision):
    """Target-layer runs longer than one multi-copy GLN launch (5:1), runs with
    no full layer after them (3:0), full-only stacks (0:1) and repeated blocks."""
    _run(_wl(K, P, blocks), 3, precision)


@pytest.mark.parametrize("per_scen", [1, 4, 16, 64])
def test_targets_per_user(per_scen):
    """4 scenarios x per_scen exposures = 4..256 targets per user: T query
    tiles from a fraction of one tile to two full tiles per scenario."""
    _run(_wl(3, 1, hist_len=40, rt_len=10, exp_per_scen=per_scen, seed=17), 2, "bf16")


@pytest.mark.parametrize("norm", ["valid", "seqlen", "none"])
def test_attn_norm(norm):
    _run(_wl(1, 1, norm=norm), 3, "bf16")


@pytest.mark.parametrize("d,H,G", [(256, 4, 2), (256, 2, 1), (512, 4, 4), (128, 8, 2)])
def test_head_dims(d, H, G):
    """Every bf16 attention specialisation (head_dim 64, 128, 128 with MHA, 16) against the
    oracle; head_dim 32 and 256 are the small / paper goldens."""
    wl = datagen.WORKLOADS["small"]()
    hta = dataclasses.replace(wl.cfg.hta, d_model=d, heads=H, kv_heads=G, target_layers=1, full_layers=1)
    cfg = dataclasses.replace(wl.cfg, hta=hta, d_expert=d)
    wl = dataclasses.replace(wl, cfg=cfg, hist_len=150, rt_len=40, exp_per_scen=3)
    _run(wl, 4, "bf16")


@pytest.mark.parametrize("n_hist,n_rt,n_scen", [(1, 0, 4), (0, 1, 2), (3, 2, 1), (2, 1, 6), (0, 0, 3)])
def test_schema_shapes(n_hist, n_rt, n_scen):
    """Token-source layouts other than the BASELINE one (2 H + 1 R sequences, 4 scenarios):
    no realtime or no historical sequence, no context at all (targets attend to themselves),
    more sequences, one or six scenarios."""
    wl = datagen.WORKLOADS["small"]()
    wl = dataclasses.replace(wl, schemas=datagen.make_schemas(n_scenarios=n_scen, n_hist=n_hist, n_rt=n_rt),
                             hist_len=50, rt_len=15, exp_per_scen=3)
    for precision in ("bf16", "fp32"):
        _run(wl, 5, precision)


def _random_case(seed):
    rng = np.random.default_rng(seed)
    d = int(rng.choice([128, 256, 512]))
    dh = int(rng.choice([16, 32, 64, 128]))
    dh = min(dh, d)
    H = d // dh
    G = int(rng.choice([g for g in (1, 2, 4, H) if H % g == 0]))
    K, P = [(0, 1), (1, 1), (2, 1), (3, 0), (1, 2), (3, 1)][int(rng.integers(6))]
    blocks = int(rng.integers(1, 3))
    norm = str(rng.choice(["valid", "none", "seqlen"]))
    wl = datagen.WORKLOADS["small"]()
    hta = dataclasses.replace(wl.cfg.hta, d_model=d, heads=H, kv_heads=G, target_layers=K, full_layers=P,
                              blocks=blocks, norm=norm)
    cfg = dataclasses.replace(wl.cfg, hta=hta, d_expert=int(rng.choice([64, 128, d])), experts=int(rng.integers(2, 5)))
    schemas = datagen.make_schemas(n_scenarios=int(rng.integers(1, 5)), n_hist=int(rng.integers(0, 3)),
                                   n_rt=int(rng.integers(0, 2)))
    return dataclasses.replace(wl, cfg=cfg, schemas=schemas, seed=seed,
                               hist_len=("lognormal", 40, 1.0, 0, 300), rt_len=("lognormal", 10, 1.0, 0, 80),
                               exp_per_scen=("lognormal", 4, 1.0, 1, 24))


@pytest.mark.parametrize("seed", range(40))
def test_random_configs(seed):
    """Seeded random model geometries (d, head_dim, GQA ratio, layer mix, blocks, row
    norm, experts, d_expert) and token-source layouts with heavy-tailed ragged users,
    in bf16 and fp32 check mode, against the oracle."""
    wl = _random_case(seed)
    for precision in ("bf16", "fp32"):
        _run(wl, 6, precision)
