"""GPU parity: the sm_100a solver against the CPU oracle, bit for bit.

Re-expresses the reference hot-path tests through the C-ABI
(paper_2306_09427_b200 -> include/fibra_cuda.h):
  * batch == sequential bitwise on sigma, C, u, v, f_int      test_batch.cpp:134-178
  * failed points listed individually                          test_batch.cpp:180-190
  * identity converges in 0 iterations, iteration cap          test_relax.cpp:51-69
  * warm start from the solution <= 2 iterations               test_relax.cpp:165-173
  * fixed DOFs frozen, fixed v = a = 0                         test_relax.cpp:152-163
  * solves == 7 per point with the tangent                     test_batch.cpp:222-245
plus iteration counts and full PackedStates bitwise against the oracle.
"""
import numpy as np
import pytest

import oracle as O
import paper_2306_09427_b200 as P
from _pairs import batch_F, knn, oracle_batch, same_bits

pytestmark = pytest.mark.gpu

STATE_KEYS = ("u", "v", "a", "f_int", "f_damp", "mass", "inv_mass", "t", "iters", "converged")


def gpu_batch(pnets, eop, F, relax=None, law=None, tangent=True, stiff=None, states=None):
    lib = P.RveLibrary(list(pnets), policy="explicit", explicit_assignment=list(eop))
    st, assign = P.init_batch(np.zeros(len(eop), np.int32), lib, 0)
    if states is not None:
        st = states
    br = P.batch_response(lib, assign, st, law or P.FiberLaw(), F, relax or P.RelaxConfig(),
                          stiff or P.StiffnessConfig(), want_tangent=tangent)
    return br, st


def check_states(gst, ost, keys=STATE_KEYS):
    for k in keys:
        g = getattr(gst, k)
        o = ost.arrays[k]
        assert g.shape == o.shape, k
        assert same_bits(g, o), f"state array {k} differs"


@pytest.fixture(scope="module")
def small_lib(oracle_lib):
    # test_batch.cpp:17-29 library
    a = knn(14, 38, 101, neighbors=9)
    b = knn(12, 32, 102, neighbors=9)
    return [a[0], b[0]], [a[1], b[1]]


def test_single_rve_stress_bitwise(oracle_lib):
    pn, on = knn(20, 56, 31)
    F = np.diag([1.06, 1.0, 0.97])[None]
    br, gst = gpu_batch([pn], [0], F, tangent=False)
    resp, status, ost = oracle_batch([on], [0], F, tangent=False, threads=1)
    assert status[0] == 0 and br.failed == []
    rec = br.records[0]
    assert rec["base_report"]["iterations"] == resp[0]["base_report"]["iterations"] > 0
    for k in ("residual", "eps_eff", "kinetic_fraction", "dt"):
        assert same_bits(rec["base_report"][k], resp[0]["base_report"][k]), k
    assert same_bits(rec["sigma"], resp[0]["sigma"])
    assert same_bits(rec["pk2"], resp[0]["pk2"])
    assert same_bits(rec["stress_asymmetry"], resp[0]["stress_asymmetry"])
    check_states(gst, ost)


def test_config1_batch_stress_bitwise(oracle_lib):
    pn, on = knn(375, 1000, 1)
    F = batch_F(8)
    br, gst = gpu_batch([pn], [0] * 8, F, tangent=False)
    resp, status, ost = oracle_batch([on], [0] * 8, F, tangent=False)
    assert list(np.nonzero(status)[0]) == br.failed
    for p in range(8):
        r = br.records[p]
        assert r["base_report"]["iterations"] == resp[p]["base_report"]["iterations"]
        assert same_bits(r["sigma"], resp[p]["sigma"])
        assert same_bits(r["base_report"]["residual"], resp[p]["base_report"]["residual"])
    check_states(gst, ost)


def test_batch_tangent_bitwise(small_lib):
    pnets, onets = small_lib
    lib = P.RveLibrary(pnets)
    st, assign = P.init_batch(np.zeros(8, np.int32), lib, 7)
    F = batch_F(8)
    br = P.batch_response(lib, assign, st, P.FiberLaw(), F, P.RelaxConfig(), P.StiffnessConfig())
    resp, status, ost = oracle_batch(onets, assign.entry_of_point, F, tangent=True)
    assert br.failed == [] and not status.any()
    for p in range(8):
        assert same_bits(br.responses[p].sigma, resp[p]["sigma"])
        assert same_bits(br.responses[p].spatial_c, resp[p]["spatial_c"])
        assert same_bits(br.records[p]["material_a"].reshape(6, 6), resp[p]["material_a"])
        assert br.stats[p].solves == 7
        assert br.stats[p].relax_iterations == resp[p]["relax_iterations"]
    check_states(st, ost)


def test_schedule_modes_bitwise(small_lib):
    """The start order of base solves (and the completion-order probe FIFO) changes nothing:
    batch order, strain order and a caller hint give identical records and states, with a
    failed point (collapse) and a kinematics failure mixed in."""
    pnets, _ = small_lib
    lib = P.RveLibrary(pnets)
    n = 40
    F = batch_F(n)
    F[5] = np.diag([1e-9, 1e-9, 1e-9])
    F[17] = np.diag([-1.0, 1.0, 1.0])
    F[23] = np.eye(3)
    outs = []
    for mode, hint in ((P.SCHED_BATCH, None), (P.SCHED_STRAIN, None),
                       (P.SCHED_HINT, np.arange(n, dtype=np.float64) % 7)):
        st, assign = P.init_batch(np.zeros(n, np.int32), lib, 3)
        db = P.DeviceBatch(lib, assign)
        db.set_schedule(mode, hint)
        rec = db.solve(F, want_tangent=True)
        db.download_states(st)
        db.close()
        outs.append((rec, st))
    r0, s0 = outs[0]
    assert sorted(np.nonzero(r0["status"])[0].tolist()) == [5, 17]
    for rec, st in outs[1:]:
        assert rec.tobytes() == r0.tobytes()
        for k in STATE_KEYS:
            assert same_bits(getattr(st, k), getattr(s0, k)), k


def test_exponential_law_bitwise(oracle_lib):
    """Exponential law on the resident kernel, bitwise: expm1 / exp on the device replay the
    host libm's sequences (csrc/libm_glibc.cuh; test_gpu_cluster.check_exponential)."""
    from test_gpu_cluster import check_exponential
    pn, on = knn(375, 1000, 1)
    F = batch_F(4)
    lib = P.RveLibrary([pn])
    st, assign = P.init_batch(np.zeros(4, np.int32), lib, 0)
    br = P.batch_response(lib, assign, st, P.FiberLaw(kind="exponential", nonlinearity=1.2), F,
                          P.RelaxConfig(), P.StiffnessConfig())
    resp, status, _ = oracle_batch([on], [0] * 4, F, tangent=True,
                                   law=O.Law(kind=1, nonlinearity=1.2))
    check_exponential(br, resp, status)


def test_buckling_off_bitwise(oracle_lib):
    """FiberLaw.buckling_off (compressed fibers carry no force, network.cpp:16-38): a
    compressive load on the resident and the cluster kernels, bitwise vs the oracle."""
    for args in ((375, 1000, 1), (712, 1900, 7)):
        pn, on = knn(*args)
        F = np.stack([np.diag([0.97, 1.01, 1.0]), np.diag([1.03, 0.96, 0.98])])
        law = P.FiberLaw(buckling_off=True)
        lib = P.RveLibrary([pn])
        st, assign = P.init_batch(np.zeros(2, np.int32), lib, 0)
        br = P.batch_response(lib, assign, st, law, F, P.RelaxConfig(), P.StiffnessConfig(),
                              want_tangent=False)
        resp, status, ost = oracle_batch([on], [0, 0], F, tangent=False,
                                         law=O.Law(buckling_off=True))
        assert br.failed == list(np.nonzero(status)[0])
        for p in range(2):
            if status[p]:
                continue
            r = br.records[p]
            assert r["base_report"]["iterations"] == resp[p]["base_report"]["iterations"]
            assert same_bits(r["sigma"], resp[p]["sigma"])
        check_states(st, ost)


def test_failed_points_reported(small_lib):
    pnets, _ = small_lib
    lib = P.RveLibrary(pnets)
    st, assign = P.init_batch(np.zeros(3, np.int32), lib, 7)
    F = np.tile(np.diag([1.02, 1.0, 1.0]), (3, 1, 1))
    # The reference test uses diag(1e-9, 1, 1); its own relax TUs converge on that load
    # (DESIGN.md "reference test discrepancies"), so squeeze every axis to collapse the
    # boundary-to-boundary fibers at the first force pass instead.
    F[1] = np.diag([1e-9, 1e-9, 1e-9])
    br = P.batch_response(lib, assign, st, P.FiberLaw(), F, P.RelaxConfig(), P.StiffnessConfig())
    assert br.failed == [1]
    assert br.records[1]["status"] == 3  # FIBRA_E_COLLAPSE
    assert br.stats[1].solves == 0 and np.all(br.responses[1].sigma == 0)
    F[2] = np.diag([-1.0, 1.0, 1.0])  # det(F) <= 0 -> KinematicsError from polar_decompose
    st, assign = P.init_batch(np.zeros(3, np.int32), lib, 7)
    br = P.batch_response(lib, assign, st, P.FiberLaw(), F, P.RelaxConfig(), P.StiffnessConfig())
    assert br.failed == [1, 2] and br.records[2]["status"] == 2


def test_identity_and_iteration_cap(oracle_lib):
    pn, on = knn(16, 44, 11)
    br, _ = gpu_batch([pn], [0], np.eye(3)[None], tangent=False)
    assert br.base_reports[0]["iterations"] == 0 and br.base_reports[0]["converged"] == 1
    cfg = P.RelaxConfig(max_iterations=2)
    br, st = gpu_batch([pn], [0], np.diag([1.3, 1, 1])[None], relax=cfg, tangent=False)
    assert br.failed == [0]  # base not converged -> SolverError -> failed
    assert st.iters[0] == 2 and st.converged[0] == 0
    o = O.State(on.n_dof, on.n_free)
    _, rep = O.relax_solve(on, np.diag([1.3, 1, 1]), O.RelaxConfig(max_iterations=2), state=o)
    assert same_bits(st.u, o.u) and same_bits(st.v, o.v)


def test_warm_start_and_fixed_dofs(oracle_lib):
    pn, _ = knn(20, 56, 31)
    F = np.diag([1.06, 1.0, 0.97])[None]
    lib = P.RveLibrary([pn])
    st, assign = P.init_batch(np.zeros(1, np.int32), lib, 0)
    br1 = P.batch_response(lib, assign, st, P.FiberLaw(), F, P.RelaxConfig(), P.StiffnessConfig(),
                           want_tangent=False)
    it1 = br1.base_reports[0]["iterations"]
    br2 = P.batch_response(lib, assign, st, P.FiberLaw(), F, P.RelaxConfig(), P.StiffnessConfig(),
                           want_tangent=False)
    assert it1 > 0 and br2.base_reports[0]["iterations"] <= 2
    nf = pn.n_free
    assert np.all(st.v[nf:] == 0) and np.all(st.a[nf:] == 0)
    X = pn.packed_ref_coords[nf:].reshape(-1, 3)
    want = (X @ F[0].T - X).reshape(-1)
    assert np.max(np.abs(st.u[nf:] - want)) < 1e-15


def test_config1_tangent_bitwise(oracle_lib):
    pn, on = knn(375, 1000, 4)
    F = batch_F(2)
    br, gst = gpu_batch([pn], [0, 0], F, tangent=True)
    resp, status, ost = oracle_batch([on], [0, 0], F, tangent=True)
    assert br.failed == list(np.nonzero(status)[0])
    for p in range(2):
        if status[p]:
            continue
        assert same_bits(br.responses[p].sigma, resp[p]["sigma"])
        assert same_bits(br.responses[p].spatial_c, resp[p]["spatial_c"])
        assert br.stats[p].relax_iterations == resp[p]["relax_iterations"]
    check_states(gst, ost)


def test_cpp_dropin_shim_bitwise():
    """include/fibra_b200/batch_response.hpp driven by the reference's own C++ types and
    generator (tests/cpp/test_shim.cpp, built here by `make -C tests/cpp`)."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(__file__), "cpp", "build", "test_shim")
    if not os.path.exists(exe):
        pytest.skip("tests/cpp/build/test_shim not built (needs /root/reference)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout


def test_node_kernel_config1_batch_bitwise(oracle_lib, monkeypatch):
    """The opt-in node-centric kernel (FIBRA_KERNEL=node, csrc/dr_node.cuh): every fibre
    evaluated at both ends with d' = x_other - x_own, one barrier per iteration -- records
    and PackedStates bitwise against the oracle on 8 config-1 RVEs, with the tangent."""
    monkeypatch.setenv("FIBRA_KERNEL", "node")
    pn, on = knn(375, 1000, 1)
    F = batch_F(8)
    br, gst = gpu_batch([pn], [0] * 8, F, tangent=True)
    resp, status, ost = oracle_batch([on], [0] * 8, F, tangent=True)
    assert list(np.nonzero(status)[0]) == br.failed
    for p in range(8):
        if status[p]:
            continue
        r = br.records[p]
        assert r["relax_iterations"] == resp[p]["relax_iterations"]
        assert same_bits(r["sigma"], resp[p]["sigma"])
        assert same_bits(r["spatial_c"].reshape(6, 6), resp[p]["spatial_c"])
    check_states(gst, ost)
