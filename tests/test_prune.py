"""2:4 pruning: prune_model_projections (prune.hpp:92-103)
restated (oracle) and run on the device (mtfm_cuda_prune_projections), both
bit-exact against the weights the unmodified reference pruned
(tests/golden/prune_j.npz, ref_dump --prune), and the pruned model's records
against the reference's forward of the pruned model."""
import numpy as np
import pytest

import mtfm_oracle as O
from golden_util import batch, load, model, model_raw, ref_records
from helpers import from_oracle, rel_err


def _ref_pruned():
    a = load("prune_j")
    return a, {k[len("prune/param/"):]: v for k, v in a.items() if k.startswith("prune/param/")}


def test_oracle_prune_matches_reference():
    a, want = _ref_pruned()
    _, _, P = model_raw("prune_j")  # unpruned (init + jitter); the golden holds the reference's pruned copies
    groups = zeros = tail = 0
    names = [n for n in P if O.is_projection_param(n)]
    assert names == list(want)
    for n in names:
        w, z, g, t = O.prune_2_4(P[n])
        assert np.array_equal(w, want[n]), n
        zeros, groups, tail = zeros + z, groups + g, tail + t
    assert [groups, zeros, tail, len(names)] == a["prune/report"].tolist()


def _unpruned_model(precision):
    from paper_2602_11235_b200 import Model
    osch, ocfg, P = model_raw("prune_j")
    sch, cfg = from_oracle(osch, ocfg)
    return Model.build(sch, cfg, P, precision=precision), P


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_gpu_prune_bit_exact_and_scores(precision):
    a, want = _ref_pruned()
    m, P = _unpruned_model(precision)
    rep = m.prune_projections()
    assert [rep["groups_covered"], rep["zeros_written"], rep["exempt_tail_rows"], rep["pruned_params"]] == \
        a["prune/report"].tolist()
    for n, r, c in m.param_specs():
        got = m.get_param(n, r, c)
        assert np.array_equal(got, want[n] if n in want else P[n]), n
    ra = m.forward_batch(batch("prune_j"))
    keys, z64, *_ = ref_records("prune_j")
    assert np.array_equal(np.stack([ra.user_id, ra.scenario_id, ra.exposure_index, ra.task_index], 1), keys)
    z = ra.logit.astype(np.float64)
    if precision == "fp32":
        err = rel_err(z, z64, 1.0)
        print(f"pruned model, fp32: rel err {err:.3e} vs the reference's pruned forward")
        assert err <= 1e-4
    else:
        import bf16_emu
        osch, ocfg, _ = model("prune_j")
        Pp = dict(P)
        Pp.update(want)
        z_emu = np.array([r[4] for r in bf16_emu.Bf16Oracle(osch, ocfg, Pp).forward_batch(batch("prune_j"))])
        d, d_store = float(np.max(np.abs(z - z64))), float(np.max(np.abs(z_emu - z64)))
        print(f"pruned model, bf16: max |dz| {d:.3e} (bf16 storage alone {d_store:.3e})")
        assert d <= 2 * d_store + 2e-2


@pytest.mark.gpu
def test_gpu_prune_exempts_partial_groups():
    """d = 38 (fp32 check mode, head_dim 19): every projection has 38 input rows, so two
    trailing rows per matrix are exempt (prune.hpp:42-43)."""
    from paper_2602_11235_b200 import Model, datagen
    from paper_2602_11235_b200.schema import HTAConfig, ModelConfig
    cfg = ModelConfig(HTAConfig(d_model=38, blocks=1, target_layers=1, full_layers=1, heads=2, kv_heads=1),
                      d_emb=8, experts=2, d_expert=16)
    sch = datagen.make_schemas()
    m = Model(sch, cfg, precision="fp32")
    P = datagen.random_params(m.param_specs(), seed=11)
    m.set_params(P)
    rep = m.prune_projections()
    names = [n for n, _, _ in m.param_specs() if O.is_projection_param(n)]
    exp_tail = 0
    for n in names:
        w, _, _, t = O.prune_2_4(P[n])
        exp_tail += t
        assert np.array_equal(m.get_param(n, *P[n].shape), w), n
    assert rep["exempt_tail_rows"] == exp_tail == 2 * len(names)
