"""CPU, world_size 2 over gloo: the multi-GPU host logic (shard cut + record all-gather).
The same code runs over NCCL on B200s in bench.py under torchrun."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2306_09427_b200.shard import shard_ranges


def test_shard_ranges_balance_and_cover():
    rng = np.random.default_rng(0)
    w = rng.integers(500, 5001, size=1000)
    for world in (1, 2, 4, 8):
        rr = shard_ranges(w, world)
        assert rr[0][0] == 0 and rr[-1][1] == len(w)
        assert all(rr[i][1] == rr[i + 1][0] for i in range(world - 1))
        loads = [w[lo:hi].sum() for lo, hi in rr]
        assert max(loads) - min(loads) <= 2 * w.max()


def test_plan_shards_lpt():
    """plan_shards (fibra_plan_shards): every point once, longest-processing-time balance
    (max load <= mean + largest cost), deterministic."""
    from paper_2306_09427_b200.shard import plan_shards
    rng = np.random.default_rng(1)
    c = rng.lognormal(0, 1.5, size=2000)
    for world in (1, 2, 4, 8):
        sh = plan_shards(c, world)
        allp = np.sort(np.concatenate(sh))
        assert np.array_equal(allp, np.arange(len(c)))
        loads = [c[s].sum() for s in sh]
        assert max(loads) <= c.sum() / world + c.max() + 1e-9
        assert all(np.array_equal(a, b) for a, b in zip(sh, plan_shards(c, world)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    import paper_2306_09427_b200 as P
    from paper_2306_09427_b200.shard import allgather_records
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 37
    rr = shard_ranges(np.ones(n), world)
    lo, hi = rr[rank]
    rec = np.zeros(hi - lo, P.RESULT_DTYPE)
    rec["status"] = np.arange(lo, hi)
    rec["sigma"][:, 0] = np.arange(lo, hi) * 0.5
    full = allgather_records(rec, [b - a for a, b in rr])
    # planned (non-contiguous) shards: records come back in point order
    from paper_2306_09427_b200.shard import allgather_records_planned, plan_shards
    sh = plan_shards(np.arange(n, dtype=float) % 7 + 1, world)
    mine = np.zeros(len(sh[rank]), P.RESULT_DTYPE)
    mine["status"] = sh[rank]
    planned = allgather_records_planned(mine, sh)
    assert planned["status"].tolist() == list(range(n))
    q.put((rank, full["status"].tolist(), full["sigma"][:, 0].tolist()))
    dist.destroy_process_group()


def test_allgather_records_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, status, sig in res:
        assert status == list(range(37))
        assert sig == [0.5 * i for i in range(37)]
