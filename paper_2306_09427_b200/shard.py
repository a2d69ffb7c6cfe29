"""Multi-GPU sharding of a batch of RVE points.

RVEs are independent (reference batch.cpp:169-182).  Two ways to spread a batch:
  * one process over several GPUs: DeviceBatch(devices=[...]) / fibra_cuda_open_devices,
    where the library shards the points itself and returns the records with one
    ncclAllGather (the product path of the C++ drop-in and NetworkBatchProvider);
  * one process per GPU (torchrun): every rank computes the same plan with
    ``plan_shards`` (longest-processing-time on a per-point cost, the library's own
    fibra_plan_shards), solves its points and ``allgather_records`` returns the records in
    point order to every rank (one all-gather over NCCL/NVLink; gloo on CPU).
No collective runs inside a solve.
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


def plan_shards(costs, world: int):
    """Points of each rank: longest-processing-time on `costs` (descending cost, each point
    to the least-loaded rank, ties to the lower rank), the same plan on every rank; each
    rank's points ascending."""
    import ctypes as C
    from . import _capi
    c = np.ascontiguousarray(costs, dtype=np.float64)
    dev = np.zeros(max(len(c), 1), np.int32)
    rc = _capi.load().fibra_plan_shards(c.ctypes.data_as(_capi._dp), len(c), int(world),
                                        dev.ctypes.data_as(_capi._ip))
    if rc:
        raise ValueError("fibra_plan_shards failed")
    dev = dev[:len(c)]
    del C
    return [np.nonzero(dev == r)[0].astype(np.int32) for r in range(world)]


def network_cost(net) -> float:
    """The library's schedule cost model of one network (fibra_network_cost)."""
    import ctypes as C
    from . import _capi
    v = C.c_double()
    if _capi.load().fibra_network_cost(net.desc(), C.byref(v)):
        raise ValueError("fibra_network_cost failed")
    return v.value


def allgather_records_planned(local: np.ndarray, shards, device=None):
    """All-gather of per-rank records whose points are the index lists `shards` (from
    plan_shards): one all-gather, then the records in point order."""
    full = allgather_records(local, [len(s) for s in shards], device)
    out = np.zeros(sum(len(s) for s in shards), dtype=local.dtype)
    out[np.concatenate(shards)] = full
    return out


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
