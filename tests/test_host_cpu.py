"""Host-side logic on CPU: the parameter registry mirror, the packed batch /
parameter files, and the reference CPU path reading them (the bench's CPU arm
scores the GPU arm's own bytes)."""
import json
import os
import subprocess

import numpy as np
import pytest

from golden_util import NAMES, batch, model
from helpers import from_oracle
from paper_2602_11235_b200 import datagen, packed_io
from paper_2602_11235_b200.schema import param_specs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_BENCH = os.path.join(ROOT, "oracle", "_ref", "ref_bench")


@pytest.mark.parametrize("name", NAMES)
def test_param_specs_match_reference_registration(name):
    """schema.param_specs == Model::register_params (model.hpp:377-463), through
    the pinned init port's name list and shapes."""
    osch, ocfg, P = model(name)
    sch, cfg = from_oracle(osch, ocfg)
    sp = param_specs(sch, cfg)
    assert [n for n, _, _ in sp] == list(P)
    assert all(P[n].shape == (r, c) for n, r, c in sp)


def test_packed_file_roundtrip(tmp_path):
    wl = datagen.WORKLOADS["base"]()
    b = datagen.generate(wl, n_users=24)
    p = str(tmp_path / "b.bin")
    packed_io.save_packed(p, b, wl.schemas, wl.cfg)
    b2, sch, cfg = packed_io.load_packed(p)
    assert sch == wl.schemas and cfg == wl.cfg
    for k in b:
        assert b2[k].dtype == np.asarray(b[k]).dtype or np.array_equal(b2[k], b[k])
        assert np.array_equal(b2[k], b[k]), k
    P = datagen.random_params(param_specs(wl.schemas, wl.cfg), seed=3)
    pp = str(tmp_path / "p.bin")
    packed_io.save_params(pp, P)
    P2 = packed_io.load_params(pp)
    assert list(P2) == list(P) and all(np.array_equal(P[k], P2[k]) for k in P)


@pytest.mark.skipif(not os.path.exists(REF_BENCH), reason="oracle/_ref not built")
def test_reference_reads_packed_batch(tmp_path):
    """The compiled reference scores an MTFMPB1 batch: same users, targets and
    records as the packed arrays say (records = sum of task counts)."""
    osch, ocfg, P = model("tiny")
    sch, cfg = from_oracle(osch, ocfg)
    b = batch("tiny")
    bp, pp = str(tmp_path / "b.bin"), str(tmp_path / "p.bin")
    packed_io.save_packed(bp, b, sch, cfg)
    packed_io.save_params(pp, P)
    out = subprocess.run([REF_BENCH, "--batch", bp, "--params", pp, "--threads", "2"], capture_output=True,
                         text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    r = json.loads(out.stdout.strip().splitlines()[-1])
    ntasks = {s.scenario_id: len(s.tasks) for s in sch.scenarios}
    assert r["users"] == len(b["user_id"]) and r["targets"] == len(b["exp_ts"])
    assert r["records"] == sum(ntasks[int(s)] for s in b["exp_scenario"])
