"""Multi-rank host logic on CPU (gloo, world_size 2): users are sharded with
no data-path collective; each rank's shard re-packs exactly its users, the
union of the shards' oracle records equals the full batch's records, and the
per-rank device times are combined as a max (bench.py contract)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import mtfm_oracle as O
from golden_util import batch, model
from paper_2602_11235_b200 import datagen
from paper_2602_11235_b200.shard import shard_plan, take_users


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b = batch("tiny")
    sch, cfg, P = model("tiny")
    plan = shard_plan(b, world)
    mine = take_users(b, plan[rank])
    recs = O.Oracle(sch, cfg, P).forward_batch(mine)
    keys = [r[:4] for r in recs]
    gathered = [None] * world
    dist.all_gather_object(gathered, keys)
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put((gathered, float(t.item())))
    dist.destroy_process_group()


def test_two_rank_sharding_covers_every_record():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 2.0
    sch, cfg, P = model("tiny")
    full = {tuple(r[:4]) for r in O.Oracle(sch, cfg, P).forward_batch(batch("tiny"))}
    union = [tuple(k) for part in gathered for k in part]
    assert len(union) == len(full) and set(union) == full


def test_take_users_roundtrip_and_lpt_balance():
    wl = datagen.WORKLOADS["base"]()
    b = datagen.generate(wl, n_users=64)
    plan = shard_plan(b, 4)
    assert sorted(np.concatenate(plan).tolist()) == list(range(64))
    from paper_2602_11235_b200.shard import user_costs
    c = user_costs(b)
    loads = [c[p].sum() for p in plan]
    assert max(loads) / min(loads) < 1.15  # heavy-tailed lengths, still balanced
    sub = take_users(b, plan[1])
    # every user of the shard re-packed verbatim
    for k, u in enumerate(plan[1]):
        s0, s1 = b["seq_off"][u], b["seq_off"][u + 1]
        t0, t1 = sub["seq_off"][k], sub["seq_off"][k + 1]
        e0, e1 = b["ev_off"][s0], b["ev_off"][s1]
        f0, f1 = sub["ev_off"][t0], sub["ev_off"][t1]
        assert np.array_equal(b["ev_ts"][e0:e1], sub["ev_ts"][f0:f1])
        x0, x1 = b["exp_off"][u], b["exp_off"][u + 1]
        y0, y1 = sub["exp_off"][k], sub["exp_off"][k + 1]
        assert np.array_equal(b["exp_scenario"][x0:x1], sub["exp_scenario"][y0:y1])


def test_visible_keys_match_reference_valid_counts():
    """shard.visible_keys (the LPT cost's attention term) sums exactly the
    reference's row_valid_counts (mask.hpp:35-40) over context / T rows."""
    from golden_util import load
    from paper_2602_11235_b200.shard import visible_keys
    for name in ("tiny", "small4"):
        a = load(name)
        c_ctx, c_t = visible_keys(batch(name))
        off, bounds, vc = a["plan/off"], a["plan/bounds"], a["plan/valid_count"]
        for u in range(len(c_ctx)):
            lh, lr, lt = bounds[u]
            v = vc[off[u]:off[u + 1]].astype(np.int64)
            assert c_ctx[u] == v[:lh + lr].sum() and c_t[u] == v[lh + lr:].sum()


def test_lpt_cost_follows_model_config():
    """Costs scale with the model config passed in (base: d=512, (3:1)x2)."""
    from paper_2602_11235_b200.shard import user_costs
    wl = datagen.WORKLOADS["base"]()
    b = datagen.generate(wl, n_users=16)
    small = user_costs(b)
    base = user_costs(b, wl.cfg)
    assert np.all(base > 3.5 * small)


def _dp_split_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2602_11235_b200.dp import share_unique_id, split_batch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b = batch("train_b")
    from golden_util import load
    lab = load("train_b")["batch/exp_labels"]
    mine, ml = split_batch(b, lab, world, rank)
    uid = share_unique_id(bytes(range(128)) if rank == 0 else None)
    q.put((rank, [int(u) for u in mine["user_id"]], ml.tolist(), uid == bytes(range(128))))
    dist.destroy_process_group()


def test_dp_batch_split_and_id_broadcast_gloo():
    """Data-parallel training's host side (paper_2602_11235_b200/dp.py) at world size 2:
    the users and their label rows are partitioned exactly, and every rank receives
    rank 0's NCCL unique id."""
    import multiprocessing as mp
    from golden_util import load
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29000 + os.getpid() % 1000
    ps = [ctx.Process(target=_dp_split_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    b = batch("train_b")
    lab = load("train_b")["batch/exp_labels"]
    assert got[0][1] + got[1][1] == [int(u) for u in b["user_id"]]
    assert got[0][2] + got[1][2] == lab.tolist()
    assert got[0][3] and got[1][3]
