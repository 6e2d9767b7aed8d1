"""Data-parallel training across GPUs (one process per GPU): the host side.

Trainer::train_step (train.hpp:111-147) splits a minibatch over worker threads
and reduces their gradients in worker order; here the minibatch is split over
ranks (contiguous user ranges, like the reference's worker striping keeps every
user on one worker) and the library sums the ranks' gradients with one NCCL
all-reduce (mtfm_cuda_dp_init / mtfm_cuda_train_step) before the clip and Adam,
so every rank applies the identical update.

    split_batch(batch, labels, world, rank) -> (batch, labels) of this rank
    share_unique_id(id_or_none, group)      rank 0's NCCL id to every rank
                                            (torch.distributed, any backend)
"""
from __future__ import annotations

import numpy as np

from .schema import normalize_batch
from .shard import take_users


def split_batch(batch, labels, world: int, rank: int):
    """Users [rank * U / world, (rank + 1) * U / world) and their exposures' labels."""
    b = normalize_batch(batch)
    U = len(b["user_id"])
    u0, u1 = rank * U // world, (rank + 1) * U // world
    users = np.arange(u0, u1)
    x0, x1 = int(b["exp_off"][u0]), int(b["exp_off"][u1])
    lab = np.asarray(labels)
    return take_users(b, users), lab[x0:x1]


def share_unique_id(unique_id, group=None) -> bytes:
    """Broadcast rank 0's 128-byte NCCL unique id over an existing torch.distributed group."""
    import torch
    import torch.distributed as dist
    t = torch.zeros(128, dtype=torch.uint8)
    if dist.get_rank(group) == 0:
        t[:] = torch.frombuffer(bytearray(unique_id), dtype=torch.uint8)
    dist.broadcast(t, src=0, group=group)
    return bytes(t.numpy().tobytes())
