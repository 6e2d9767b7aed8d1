"""CTA-pair GEMMs (clusters of two CTAs on an m-block pair, each TMA-loading half of
every B k-block and multicasting it to both): the streamed BN = 256 projections of
d >= 512 models with more than 2 x 148 tiles run this way. The MMAs, their order and
the epilogue are those of the single-CTA schedule, so the records must be bitwise
equal with the pairs switched off (MTFM_GEMM_PAIRS=0, read once per process, hence
one subprocess per setting), and repeated forwards bitwise identical (a hand-off race
between the two CTAs' barriers would show up as run-to-run differences). The
single-CTA schedule itself is pinned to the reference at these widths by the base_j /
paper_j parity tests. Needs a B200."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_RUN = r"""
import sys
import numpy as np
from paper_2602_11235_b200 import Model, datagen
wl = datagen.WORKLOADS[sys.argv[1]]()
b = datagen.generate(wl, n_users=int(sys.argv[2]))
m = Model(wl.schemas, wl.cfg, precision="bf16")
m.set_params(datagen.random_params(m.param_specs(), seed=5))
ra = m.forward_batch(b)
z0 = ra.logit.copy()
for _ in range(3):
    assert np.array_equal(m.forward_batch(b).logit, z0), "repeated forward differs"
np.save(sys.argv[3], np.stack([ra.logit, ra.probability]))
"""


def _logits(tmp_path, cfg, users, pairs):
    out = str(tmp_path / f"{cfg}_{pairs}.npy")
    env = dict(os.environ, MTFM_GEMM_PAIRS=str(pairs))
    r = subprocess.run([sys.executable, "-c", _RUN, cfg, str(users), out], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out)


@pytest.mark.parametrize("cfg,users", [("base", 96), ("paper", 12)])
def test_pairs_bitwise_equal_single_cta(tmp_path, cfg, users):
    a = _logits(tmp_path, cfg, users, 1)
    b = _logits(tmp_path, cfg, users, 0)
    assert a.shape == b.shape and a.shape[1] > 0
    assert np.all(np.isfinite(a))
    assert np.array_equal(a, b), f"max |dz| = {np.max(np.abs(a - b))}"
