"""CPU-side checks of the C ABI library: it builds, loads, exports every
symbol include/mtfm_cuda.h declares, validates configs like the reference,
and fails loudly (no CPU fallback) when no GPU is present."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "mtfm_cuda.h")).read()
    return sorted(set(re.findall(r"MTFM_API[^;(]*?\b(mtfm_(?:cuda|dataset|nccl)_\w+)\s*\(", src)))


def test_header_declares_the_abi():
    names = _declared()
    assert "mtfm_cuda_forward" in names and "mtfm_cuda_set_param" in names
    assert len(names) >= 16


def test_library_exports_every_declared_symbol():
    from paper_2602_11235_b200 import abi
    L = abi.lib()
    for n in _declared():
        assert hasattr(L, n), n
    bound = {s[0] for s in abi.SIGNATURES}
    assert set(_declared()) == bound


def test_version_string():
    from paper_2602_11235_b200 import abi
    assert b"sm_100a" in abi.lib().mtfm_cuda_version()


def _tiny():
    from paper_2602_11235_b200 import datagen
    return datagen.WORKLOADS["tiny"]()


def test_config_validation_matches_reference():
    # HTAConfig::validate (model_config.hpp:53-66) runs before any device work
    from paper_2602_11235_b200 import Model, abi
    wl = _tiny()
    wl.cfg.hta.kv_heads = 3
    with pytest.raises(abi.ConfigError, match="divisible by kv_heads"):
        Model(wl.schemas, wl.cfg)
    wl = _tiny()
    wl.cfg.hta.eps = 0.0
    with pytest.raises(abi.ConfigError, match="eps"):
        Model(wl.schemas, wl.cfg)


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2602_11235_b200 import Model, abi
    wl = _tiny()
    with pytest.raises(abi.MtfmError):
        Model(wl.schemas, wl.cfg)


def test_pack_samples_layout():
    from paper_2602_11235_b200 import BehaviorEvent, Exposure, SequenceRecord, UserSample, pack_samples
    s = UserSample(7, [SequenceRecord(0, [BehaviorEvent([1, 2], 10), BehaviorEvent([3, 0], 20)])],
                   [SequenceRecord(0, [BehaviorEvent([2, 4], 900)])],
                   [Exposure(1, [2], [0, 4], [3], 1100)])
    b = pack_samples([s])
    assert b["seq_off"].tolist() == [0, 2] and b["seq_kind"].tolist() == [0, 1]
    assert b["ev_off"].tolist() == [0, 2, 3] and b["ev_feats"].tolist() == [1, 2, 3, 0, 2, 4]
    assert b["exp_blk"].tolist() == [1, 2, 1] and b["exp_feats"].tolist() == [2, 0, 4, 3]


def test_datagen_shapes():
    from paper_2602_11235_b200 import datagen
    wl = datagen.WORKLOADS["small"]()
    b = datagen.generate(wl, n_users=16)
    assert len(b["ev_ts"]) == 16 * 512 and len(b["exp_ts"]) == 16 * 32
    # every sequence time-sorted
    for s in range(len(b["seq_kind"])):
        ts = b["ev_ts"][b["ev_off"][s]:b["ev_off"][s + 1]]
        assert (np.diff(ts) >= 0).all()
