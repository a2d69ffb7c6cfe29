"""Multi-GPU in the product (fibra_cuda_open_devices): one process, several B200s, points
sharded by longest-processing-time, records returned by one ncclAllGather.  Every record
and every state array must equal the single-GPU run bit for bit, before and after a
cost-hint re-plan that moves warm states between devices.  Skipped on a 1-GPU box."""
import numpy as np
import pytest

import paper_2306_09427_b200 as P
from _pairs import batch_F, knn, same_bits

pytestmark = pytest.mark.gpu

STATE_KEYS = ("u", "v", "a", "f_int", "f_damp", "mass", "inv_mass", "t", "iters", "converged")


def n_gpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.skipif("n_gpus() < 2")
def test_multi_device_bitwise_vs_single():
    nets = [knn(14, 38, 101, neighbors=9)[0], knn(20, 56, 31)[0], knn(375, 1000, 1)[0]]
    eop = np.array([2, 0, 1, 2, 1, 0, 2, 2, 1, 0, 2, 1], np.int32)
    n = len(eop)
    F = batch_F(n)
    lib = P.RveLibrary(nets, policy="explicit", explicit_assignment=[int(e) for e in eop])
    ndev = min(n_gpus(), 4)
    runs = {}
    for devs in ([0], list(range(ndev))):
        st, assign = P.init_batch(np.zeros(n, np.int32), lib, 0)
        recs = []
        for call in range(2):  # second call: warm start from the first (Newton-like)
            Fc = F.copy()
            Fc[:, 0, 0] += 0.003 * call
            br = P.batch_response(lib, assign, st, P.FiberLaw(), Fc, P.RelaxConfig(),
                                  P.StiffnessConfig(), devices=devs)
            recs.append(br.records.copy())
        runs[len(devs)] = (recs, st)
    (r1, s1), (rn, sn) = runs[1], runs[ndev]
    for a, b in zip(r1, rn):
        assert a.tobytes() == b.tobytes()
    for k in STATE_KEYS:
        assert same_bits(getattr(s1, k), getattr(sn, k)), k


@pytest.mark.skipif("n_gpus() < 2")
def test_multi_device_replan_moves_states():
    """A FIBRA_SCHED_HINT re-plan on a multi-device context moves the warm states of the
    points that change device; the next (warm-started) call equals the single-GPU one."""
    nets = [knn(20, 56, 31)[0], knn(14, 38, 101, neighbors=9)[0]]
    eop = np.array([0, 1] * 8, np.int32)
    n = len(eop)
    F = batch_F(n)
    lib = P.RveLibrary(nets, policy="explicit", explicit_assignment=[int(e) for e in eop])
    out = {}
    for devs in ([0], [0, 1]):
        assign = P.BatchAssignment(eop)
        db = P.DeviceBatch(lib, assign, devs[0], devices=devs)
        rec = db.solve(F)
        db.set_schedule(P.SCHED_HINT, np.arange(n, dtype=float)[::-1] ** 3)  # new plan
        rec2 = db.solve(F + 0.001)
        st, _ = P.init_batch(np.zeros(n, np.int32), lib, 0)
        db.download_states(st)
        out[len(devs)] = (rec.tobytes(), rec2.tobytes(), st)
        db.close()
    assert out[1][0] == out[2][0] and out[1][1] == out[2][1]
    for k in STATE_KEYS:
        assert same_bits(getattr(out[1][2], k), getattr(out[2][2], k)), k
