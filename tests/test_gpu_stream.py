"""GPU parity of the HBM-streaming kernel (csrc/dr_stream.cuh): RVEs beyond on-chip capacity,
one thread-block cluster per RVE, incidence rows streamed from HBM, x in a global double
buffer, node-centric fibre evaluation (d' = x_other - x_own), one cluster barrier per
iteration.  The same bitwise contract as tests/test_gpu_parity.py:
  * a 100k-fibre lattice (beyond a 16-CTA cluster's shared memory: the upload places it on
    the streaming kernel by itself) relaxed to convergence: iterations, sigma, PackedStates;
  * FIBRA_KERNEL=stream on config-1 RVEs with the tangent (7 solves per point);
  * the exponential law (per-pass cluster CFL minimum) and a capped config-4 lattice.
"""
import numpy as np
import pytest

import oracle as O
import paper_2306_09427_b200 as P
from _pairs import batch_F, knn, oracle_batch, same_bits
from test_gpu_cluster import check_records, check_states, lattice_pair

pytestmark = pytest.mark.gpu


def run(pnets, eop, F, tangent, relax=None, law=None):
    lib = P.RveLibrary(list(pnets), policy="explicit", explicit_assignment=list(eop))
    st, assign = P.init_batch(np.zeros(len(eop), np.int32), lib, 0)
    db = P.DeviceBatch(lib, assign)
    shapes = [db.entry_kernel(e) for e in range(len(pnets))]
    db.upload_states(st)
    rec = db.solve(F, law or P.FiberLaw(), relax or P.RelaxConfig(), P.StiffnessConfig(),
                   tangent)
    db.download_states(st)
    db.close()
    return P._to_result(rec), st, shapes


def test_stream_100k_fibre_lattice_converged(oracle_lib):
    """29^3 nodes, 100k fibres: no resident shape and no 16-CTA cluster holds it."""
    pn, on = lattice_pair(29, 100000, 3)
    F = batch_F(1)
    br, st, shapes = run([pn], [0], F, tangent=False)
    assert shapes[0]["fibers_per_thread"] == -1 and shapes[0]["cluster"] >= 2, shapes
    resp, status, ost = oracle_batch([on], [0], F, tangent=False)
    assert status[0] == 0 and br.failed == []
    assert br.records[0]["base_report"]["iterations"] == resp[0]["base_report"]["iterations"] > 0
    check_records(br, resp, status, tangent=False)
    check_states(st, ost)


def test_stream_forced_config1_tangent(oracle_lib, monkeypatch):
    monkeypatch.setenv("FIBRA_KERNEL", "stream")
    pn, on = knn(375, 1000, 1)
    F = batch_F(4)
    br, st, shapes = run([pn], [0] * 4, F, tangent=True)
    assert shapes[0]["fibers_per_thread"] == -1
    resp, status, ost = oracle_batch([on], [0] * 4, F, tangent=True)
    check_records(br, resp, status, tangent=True)
    check_states(st, ost, points=[p for p in range(4) if not status[p]])


def test_stream_exponential_law(oracle_lib, monkeypatch):
    monkeypatch.setenv("FIBRA_KERNEL", "stream")
    pn, on = knn(20, 56, 31)
    F = batch_F(3)
    law = P.FiberLaw(kind="exponential", nonlinearity=4.0)
    br, st, shapes = run([pn], [0] * 3, F, tangent=True, law=law)
    resp, status, ost = oracle_batch([on], [0] * 3, F, tangent=True,
                                     law=O.Law(kind=1, nonlinearity=4.0))
    check_records(br, resp, status, tangent=True)  # bitwise: csrc/libm_glibc.cuh


def test_stream_config4_lattice_capped(oracle_lib, monkeypatch):
    monkeypatch.setenv("FIBRA_KERNEL", "stream")
    pn, on = lattice_pair(23, 50000, 1)
    F = batch_F(2)
    relax = P.RelaxConfig(max_iterations=300)
    br, st, shapes = run([pn], [0, 0], F, tangent=False, relax=relax)
    resp, status, ost = oracle_batch([on], [0, 0], F, tangent=False,
                                     relax=O.RelaxConfig(max_iterations=300))
    assert list(status) == [6, 6] and br.failed == [0, 1]
    check_states(st, ost)
