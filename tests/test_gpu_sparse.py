"""2:4 sparse tensor cores for the pruned projections (SURVEY §8 f-4,
include/mtfm_cuda.h mtfm_cuda_set_sparse_mma): after prune_projections
(prune.hpp:92-103) the bf16 forward runs f1/fuq/fkv/f2 as tcgen05.mma.sp on the
compressed weights. Checked against the dense tensor-core path on the same
pruned weights and against the oracle's forward of the pruned model. Needs a B200."""
import dataclasses

import numpy as np
import pytest

import mtfm_oracle as O
from helpers import oracle_records, to_oracle
from paper_2602_11235_b200 import Model, abi, datagen
from paper_2602_11235_b200.schema import param_specs

pytestmark = pytest.mark.gpu


def _case(name, users, seed=3):
    wl = dataclasses.replace(datagen.WORKLOADS[name](), seed=seed)
    b = datagen.generate(wl, n_users=users)
    P = datagen.random_params(param_specs(wl.schemas, wl.cfg), seed=seed + 1)
    return wl, b, P


def test_sparse_mode_follows_the_weights():
    wl, b, P = _case("small", 2)
    m = Model(wl.schemas, wl.cfg, precision="bf16")
    m.set_params(P)
    assert m.set_sparse_mma(2) is False  # dense weights: not 2:4
    with pytest.raises(abi.ContractError):
        m.set_sparse_mma(1)
    m.set_sparse_mma(2)
    m.prune_projections()
    assert m.set_sparse_mma(2) is True
    assert m.set_sparse_mma(0) is False
    f = Model(wl.schemas, wl.cfg, precision="fp32")
    f.set_params(P)
    f.prune_projections()
    assert f.set_sparse_mma(2) is False  # the fp32 check mode stays dense


@pytest.mark.parametrize("name,users", [("small", 24), ("base", 6)])
def test_sparse_matches_dense_and_oracle(name, users):
    """d = 256 (K = 256, 2 x 128-K blocks) and d = 512 (16 heads: 5 feature tiles of f1,
    4 K blocks), ragged users so token tiles end part-way."""
    wl, b, P = _case(name, users)
    m = Model(wl.schemas, wl.cfg, precision="bf16")
    m.set_params(P)
    m.prune_projections()
    assert m.set_sparse_mma(2)
    sp = m.forward_batch(b)
    assert m.set_sparse_mma(0) is False
    de = m.forward_batch(b)
    assert np.array_equal(np.stack([sp.user_id, sp.scenario_id, sp.exposure_index, sp.task_index], 1),
                          np.stack([de.user_id, de.scenario_id, de.exposure_index, de.task_index], 1))
    d_sd = float(np.max(np.abs(sp.logit - de.logit)))
    Pp = {k: (O.prune_2_4(v)[0] if O.is_projection_param(k) else v) for k, v in P.items()}
    osch, ocfg = to_oracle(wl.schemas, wl.cfg)
    keys, z_ref, _ = oracle_records(osch, ocfg, Pp, b)
    d_sp, d_de = float(np.max(np.abs(sp.logit - z_ref))), float(np.max(np.abs(de.logit - z_ref)))
    print(f"{name}: sparse vs dense max |dz| {d_sd:.3e}; vs oracle: sparse {d_sp:.3e}, dense {d_de:.3e}")
    assert d_sd <= 1e-2
    assert d_sp <= 2e-2 and d_sp <= 2 * d_de + 5e-3


@pytest.mark.parametrize("seed", range(8))
def test_sparse_random_geometries(seed):
    """Seeded random geometries (tests/test_gpu_sweep.py::_random_case): the pruned model on
    the sparse tensor cores against the dense path on the same weights and the oracle."""
    from test_gpu_sweep import _random_case
    wl = _random_case(100 + seed)
    b = datagen.generate(wl, n_users=6)
    P = datagen.random_params(param_specs(wl.schemas, wl.cfg), seed=seed)
    m = Model(wl.schemas, wl.cfg, precision="bf16")
    m.set_params(P)
    m.prune_projections()
    assert m.set_sparse_mma(2)
    sp = m.forward_batch(b)
    m.set_sparse_mma(0)
    de = m.forward_batch(b)
    Pp = {k: (O.prune_2_4(v)[0] if O.is_projection_param(k) else v) for k, v in P.items()}
    osch, ocfg = to_oracle(wl.schemas, wl.cfg)
    keys, z_ref, _ = oracle_records(osch, ocfg, Pp, b)
    assert np.array_equal(np.stack([sp.user_id, sp.scenario_id, sp.exposure_index, sp.task_index], 1), keys)
    assert float(np.max(np.abs(sp.logit - de.logit))) <= 1e-2
    assert float(np.max(np.abs(sp.logit - z_ref))) <= 2e-2
