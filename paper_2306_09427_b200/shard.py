"""Multi-GPU sharding of a batch of RVE points (one process per GPU).

RVEs are independent (reference batch.cpp:169-182), so a batch is cut into contiguous
per-rank ranges balanced by a cost weight (fibers per point by default), each
rank solves its range on its own B200, and one all-gather over NCCL (NVLink) returns the
fixed-size result records to every rank.  No collective runs inside a solve.
"""
from __future__ import annotations

import numpy as np


def shard_ranges(weights, world: int):
    """Contiguous [lo, hi) per rank with near-equal cumulative weight."""
    w = np.asarray(weights, dtype=np.float64)
    n = len(w)
    if world <= 1 or n == 0:
        return [(0, n)] + [(n, n)] * max(0, world - 1)
    cum = np.concatenate([[0.0], np.cumsum(w)])
    cuts = [0]
    for r in range(1, world):
        target = cum[-1] * r / world
        cuts.append(int(np.clip(np.searchsorted(cum, target, side="left"), cuts[-1], n)))
    cuts.append(n)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def allgather_records(local: np.ndarray, counts, device=None):
    """All-gather structured result records of unequal per-rank length.

    `local` is this rank's structured array; `counts` the per-rank lengths.  Uses one
    torch.distributed.all_gather_into_tensor on bytes (NCCL on CUDA tensors, gloo on CPU).
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    item = local.dtype.itemsize
    cap = max(counts) if counts else 0
    buf = np.zeros(cap * item, np.uint8)
    raw = local.view(np.uint8).reshape(-1)
    buf[:raw.size] = raw
    t = torch.from_numpy(buf)
    if device is not None:
        t = t.to(device)
    out = torch.empty(world * cap * item, dtype=torch.uint8, device=t.device)
    dist.all_gather_into_tensor(out, t)
    host = out.cpu().numpy()
    parts = [host[r * cap * item:(r * cap + counts[r]) * item] for r in range(world)]
    return np.frombuffer(np.concatenate(parts).tobytes(), dtype=local.dtype)
