"""Training on the GPU against the reference Trainer itself:
tests/golden/train_{a,b}.npz hold, for every user of the fixture in one
minibatch, the gradients of Trainer::train_step's first step (train.hpp:111-147,
x 1/batch, before clipping), the parameters after it (ParamStore::adam_step,
params.hpp:87-119, global-norm clip 1.0) and after three steps, and the three
losses — all from the unmodified reference on its f64 path (ref_dump --train).

Tolerances (fp32 SIMT vs the reference's f64): loss <= 2e-5 relative; every
gradient tensor within 2e-4 of its largest entry (plus 1e-7); parameters after
Adam within 2e-3 * lr (Adam normalises each coordinate, so a coordinate whose
gradient is ~1e-8 can move by up to lr in either implementation: those are
allowed, counted and bounded)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from golden_util import batch, load, model
from helpers import from_oracle
from paper_2602_11235_b200 import Model

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _setup(name):
    a = load(name)
    osch, ocfg, P = model(name)
    sch, cfg = from_oracle(osch, ocfg)
    m = Model.build(sch, cfg, P, precision="fp32")
    lr, b1, b2, eps, clip, steps = (float(x) for x in a["train/cfg"])
    return a, m, P, dict(lr=lr, beta1=b1, beta2=b2, eps=eps, clip_norm=clip)


def _close_params(m, a, key, lr):
    worst, loose = 0.0, 0
    for n, r, c in m.param_specs():
        got = m.get_param(n, r, c)
        want = a[f"train/{key}/{n}"]
        d = np.abs(got - want)
        loose += int(np.sum(d > 2e-3 * lr))
        worst = max(worst, float(d.max()))
    return worst, loose


@pytest.mark.parametrize("name", ["train_a", "train_b"])
def test_train_step_matches_reference_trainer(name):
    a, m, P, cfg = _setup(name)
    b = batch(name)
    labels = a["batch/exp_labels"]
    res = m.train_step(b, labels, **cfg)
    want_loss = a["train/loss"]
    print(f"{name}: step 1 loss {res.loss:.9f} (reference {want_loss[0]:.9f}), grad norm {res.grad_norm:.6f}")
    assert abs(res.loss - want_loss[0]) <= 2e-5 * abs(want_loss[0])
    worst = 0.0
    for n, r, c in m.param_specs():
        g = m.get_grad(n, r, c)
        want = a[f"train/grad/{n}"]
        tol = 2e-4 * float(np.abs(want).max()) + 1e-7
        err = float(np.abs(g - want).max())
        worst = max(worst, err / (float(np.abs(want).max()) + 1e-12))
        assert err <= tol, (n, err, tol)
    print(f"{name}: worst gradient error / max|grad| = {worst:.3e}")
    w1, loose1 = _close_params(m, a, "param1", cfg["lr"])
    n_par = sum(r * c for _, r, c in m.param_specs())
    print(f"{name}: params after step 1: max |dw| {w1:.3e} (lr {cfg['lr']}), {loose1} of {n_par} beyond 2e-3 lr")
    assert w1 <= 2 * cfg["lr"] + 1e-6 and loose1 <= max(3, n_par // 2000)
    for k in (1, 2):
        r2 = m.train_step(b, labels, **cfg)
        print(f"{name}: step {k + 1} loss {r2.loss:.9f} (reference {want_loss[k]:.9f})")
        assert abs(r2.loss - want_loss[k]) <= 1e-4 * abs(want_loss[k])
    wN, looseN = _close_params(m, a, "paramN", cfg["lr"])
    print(f"{name}: params after 3 steps: max |dw| {wN:.3e}, {looseN} beyond 2e-3 lr")
    assert wN <= 6 * cfg["lr"] and looseN <= max(6, n_par // 1000)


def test_trained_weights_serve_and_reupload():
    """After training, the fp32 handle forwards with the new weights, and a bf16 model
    built from get_param() scores like it (parameters leave the device by name)."""
    a, m, P, cfg = _setup("train_b")
    b = batch("train_b")
    m.train_step(b, a["batch/exp_labels"], **cfg)
    z32 = m.forward_batch(b).logit
    newP = {n: m.get_param(n, r, c) for n, r, c in m.param_specs()}
    assert any(not np.array_equal(newP[n], P[n]) for n in P)
    m2 = Model.build(m.schemas, m.cfg, newP, precision="fp32")
    assert np.array_equal(m2.forward_batch(b).logit, z32)


def test_missing_label_is_integrity_error():
    from paper_2602_11235_b200 import abi
    a, m, P, cfg = _setup("train_a")
    lab = a["batch/exp_labels"].copy()
    lab[0, 0] = -1
    with pytest.raises(abi.IntegrityError):
        m.train_step(batch("train_a"), lab, **cfg)


DP_SCRIPT = r"""
import os, sys, numpy as np
sys.path[:0] = [{root!r}, {root!r} + "/tests", {root!r} + "/oracle"]
import torch, torch.distributed as dist
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
from golden_util import batch, load, model
from helpers import from_oracle
from paper_2602_11235_b200 import Model
from paper_2602_11235_b200.dp import share_unique_id, split_batch
a = load("train_b")
osch, ocfg, P = model("train_b")
sch, cfg = from_oracle(osch, ocfg)
m = Model.build(sch, cfg, P, precision="fp32", device=rank)
uid = share_unique_id(Model.nccl_unique_id() if rank == 0 else None)
m.dp_init(world, rank, uid)
b = batch("train_b")
mine, lab = split_batch(b, a["batch/exp_labels"], world, rank)
lr, b1, b2, eps, clip, _ = (float(x) for x in a["train/cfg"])
for _ in range(3):
    r = m.train_step(mine, lab, lr=lr, beta1=b1, beta2=b2, eps=eps, clip_norm=clip, global_batch=len(b["user_id"]))
W = np.concatenate([m.get_param(n, rr, cc).ravel() for n, rr, cc in m.param_specs()])
np.save(sys.argv[1] + f"_{{rank}}.npy", W)
np.save(sys.argv[1] + f"_loss_{{rank}}.npy", np.array([r.loss]))
dist.destroy_process_group()
"""


def test_data_parallel_two_gpus_equals_one(tmp_path):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (gpurun --gpus 2)")
    a, m, P, cfg = _setup("train_b")
    b = batch("train_b")
    for _ in range(3):
        r1 = m.train_step(b, a["batch/exp_labels"], **cfg)
    W1 = np.concatenate([m.get_param(n, rr, cc).ravel() for n, rr, cc in m.param_specs()])
    out = str(tmp_path / "dp")
    script = tmp_path / "dp.py"
    script.write_text(DP_SCRIPT.format(root=ROOT))
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29561")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", "29561", str(script), out]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    W0, Wr = np.load(out + "_0.npy"), np.load(out + "_1.npy")
    assert np.array_equal(W0, Wr), "ranks diverged"
    l0 = float(np.load(out + "_loss_0.npy")[0])
    print(f"dp: 3 steps on 2 GPUs, max |W_dp - W_1gpu| = {np.abs(W0 - W1).max():.3e}, loss {l0:.9f} vs {r1.loss:.9f}")
    assert np.abs(W0 - W1).max() <= 2e-3 * cfg["lr"] * 3 + 1e-6
    assert abs(l0 - r1.loss) <= 1e-5 * abs(r1.loss)
