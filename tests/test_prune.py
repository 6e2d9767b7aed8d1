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


def test_prune_restatement_exempts_partial_groups_and_ties():
    """prune.hpp:42-66 on hand-checkable input: a 6-row matrix has one full group and two
    exempt tail rows; equal magnitudes keep the earlier rows."""
    w = np.array([[1, -3, 2], [-4, 3, 2], [2, 1, 2], [3, 0, 2], [9, 9, 9], [-9, 9, 9]], np.float32)
    got, zeros, groups, tail = O.prune_2_4(w)
    want = np.array([[0, -3, 2], [-4, 3, 2], [0, 0, 0], [3, 0, 0], [9, 9, 9], [-9, 9, 9]], np.float32)
    assert np.array_equal(got, want) and (zeros, groups, tail) == (6, 3, 2)
