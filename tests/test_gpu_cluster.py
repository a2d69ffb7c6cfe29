"""GPU parity of the cluster kernel: RVEs too large for one CTA.

The same bitwise contract as tests/test_gpu_parity.py (iterations, sigma, C and the whole
PackedStates equal to the oracle's bits), for networks that upload_library places on a
thread-block cluster (csrc/dr_cluster.cuh, host/cluster_schedule.cpp):
  * stress-only batch on a ~1.9k-fiber knn network (2-CTA cluster), natural convergence;
  * a mixed library (resident entry + cluster entry) with the tangent (7 solves/point);
  * the exponential law (per-pass cluster CFL minimum);
  * a config-3-sized 5k-fiber network under an iteration cap (state after the cap);
  * identity (0 iterations) and a collapsing point on the cluster path.
"""
import numpy as np
import pytest

import oracle as O
import paper_2306_09427_b200 as P
from _pairs import batch_F, knn, oracle_batch, same_bits

pytestmark = pytest.mark.gpu

STATE_KEYS = ("u", "v", "a", "f_int", "f_damp", "mass", "inv_mass", "t", "iters", "converged")


def check_states(gst, ost, points=None):
    """PackedStates bitwise; `points` restricts the check (a solve that throws leaves a
    half-written state in the reference, which is not mirrored -- DESIGN.md)."""
    if points is None:
        for k in STATE_KEYS:
            assert same_bits(getattr(gst, k), ost.arrays[k]), f"state array {k} differs"
        return
    nd = np.diff(np.asarray(gst.offsets))
    for p in points:
        lo, hi = int(gst.offsets[p]), int(gst.offsets[p + 1])
        for k in STATE_KEYS:
            g, o = getattr(gst, k), ost.arrays[k]
            sl = slice(p, p + 1) if len(g) == len(nd) else slice(lo, hi)
            assert same_bits(g[sl], o[sl]), f"point {p}: state array {k} differs"


def run(pnets, eop, F, tangent, relax=None, law=None, force_cluster=None):
    """batch_response on the GPU; `force_cluster` = C puts every entry on a C-CTA cluster
    (FIBRA_FORCE_CLUSTER) -- networks up to ~2.5k fibres would otherwise run resident."""
    import os
    old = os.environ.get("FIBRA_FORCE_CLUSTER")
    if force_cluster:
        os.environ["FIBRA_FORCE_CLUSTER"] = str(force_cluster)
    try:
        return _run(pnets, eop, F, tangent, relax, law)
    finally:
        if force_cluster:
            if old is None:
                del os.environ["FIBRA_FORCE_CLUSTER"]
            else:
                os.environ["FIBRA_FORCE_CLUSTER"] = old


def _run(pnets, eop, F, tangent, relax=None, law=None):
    lib = P.RveLibrary(list(pnets), policy="explicit", explicit_assignment=list(eop))
    st, assign = P.init_batch(np.zeros(len(eop), np.int32), lib, 0)
    db = P.DeviceBatch(lib, assign)
    shapes = [db.entry_kernel(i) for i in range(len(pnets))]
    db.close()
    br = P.batch_response(lib, assign, st, law or P.FiberLaw(), F, relax or P.RelaxConfig(),
                          P.StiffnessConfig(), want_tangent=tangent)
    return br, st, shapes


def check_records(br, resp, status, tangent):
    assert br.failed == list(np.nonzero(status)[0])
    for p, r in enumerate(br.records):
        if status[p]:
            assert r["status"] == status[p]
            continue
        o = resp[p]
        assert r["base_report"]["iterations"] == o["base_report"]["iterations"]
        for k in ("residual", "eps_eff", "kinetic_fraction", "dt"):
            assert same_bits(r["base_report"][k], o["base_report"][k]), (p, k)
        assert same_bits(r["sigma"], o["sigma"]), p
        assert same_bits(r["pk2"], o["pk2"]), p
        if tangent:
            assert same_bits(r["spatial_c"].reshape(6, 6), o["spatial_c"]), p
            assert r["relax_iterations"] == o["relax_iterations"]


@pytest.fixture(scope="module")
def mid_net(oracle_lib):
    return knn(712, 1900, 7)


def test_cluster_stress_bitwise(mid_net):
    pn, on = mid_net
    F = batch_F(6)
    br, st, shapes = run([pn], [0] * 6, F, tangent=False, force_cluster=2)
    assert shapes[0]["cluster"] == 2
    resp, status, ost = oracle_batch([on], [0] * 6, F, tangent=False)
    check_records(br, resp, status, tangent=False)
    check_states(st, ost)


def test_cluster_2500_fibers_bitwise(oracle_lib):
    """A config-3 size between the shapes (2.5k fibers: 2 CTAs of the (384, 4, 1) shape)."""
    pn, on = knn(625, 2500, 11)
    F = batch_F(4)
    br, st, shapes = run([pn], [0] * 4, F, tangent=False, force_cluster=2)
    assert shapes[0]["cluster"] == 2 and shapes[0]["fibers_per_thread"] == 4
    resp, status, ost = oracle_batch([on], [0] * 4, F, tangent=False)
    check_records(br, resp, status, tangent=False)
    check_states(st, ost)


def test_cluster_tangent_mixed_library(oracle_lib):
    pn, on = lattice_pair(12, 6000, 5)  # beyond the resident shapes: a cluster entry
    sp, so = knn(14, 38, 101, neighbors=9)
    F = batch_F(4)
    eop = [1, 0, 1, 0]
    br, st, shapes = run([sp, pn], eop, F, tangent=True)
    assert shapes[0]["cluster"] == 1 and shapes[1]["cluster"] >= 2
    resp, status, ost = oracle_batch([so, on], eop, F, tangent=True)
    check_records(br, resp, status, tangent=True)
    check_states(st, ost)


def check_exponential(br, resp, status):
    """Exponential law: the device evaluates expm1 / exp with the host libm's own operation
    sequences (csrc/libm_glibc.cuh), so the contract is bitwise like the linear law's:
    iteration counts, sigma and the tangent."""
    check_records(br, resp, status, tangent=True)


def test_cluster_exponential_law(mid_net):
    pn, on = mid_net
    F = batch_F(3)
    law = P.FiberLaw(kind="exponential", nonlinearity=4.0)
    br, st, shapes = run([pn], [0] * 3, F, tangent=True, law=law, force_cluster=2)
    assert shapes[0]["cluster"] >= 2
    resp, status, ost = oracle_batch([on], [0] * 3, F, tangent=True,
                                     law=O.Law(kind=1, nonlinearity=4.0))
    check_exponential(br, resp, status)


def test_cluster_config3_size_capped(oracle_lib):
    pn, on = knn(1250, 5000, 3)  # config 3's largest size (N = M / 4)
    F = batch_F(2)
    relax = P.RelaxConfig(max_iterations=3000)
    br, st, shapes = run([pn], [0, 0], F, tangent=False, relax=relax)
    assert shapes[0]["cluster"] >= 2
    resp, status, ost = oracle_batch([on], [0, 0], F, tangent=False,
                                     relax=O.RelaxConfig(max_iterations=3000))
    assert list(status) == [6, 6]  # not converged within the cap -> failed, as the reference
    assert br.failed == [0, 1]
    check_states(st, ost)


def test_cluster_identity_and_collapse(mid_net):
    pn, on = mid_net
    F = np.stack([np.eye(3), np.diag([1e-9, 1e-9, 1e-9]), batch_F(1)[0]])
    br, st, _ = run([pn], [0] * 3, F, tangent=False, force_cluster=2)
    resp, status, ost = oracle_batch([on], [0] * 3, F, tangent=False)
    assert br.records[0]["base_report"]["iterations"] == 0
    assert br.records[1]["status"] == 3 and status[1] == 3
    check_records(br, resp, status, tangent=False)
    check_states(st, ost, points=[0, 2])


def lattice_pair(n, m, seed):
    pn = P.generate_lattice_network(n, m, seed)
    on = O.Network(pn.coords, pn.fiber_nodes[:, 0], pn.fiber_nodes[:, 1], pn.fiber_area,
                   pn.fiber_modulus, pn.box_half)
    return pn, on


def test_cluster_config4_lattice_capped(oracle_lib):
    """A config-4 sized RVE (50k fibers, 12.2k nodes) on a 16-CTA cluster: the full state
    after an iteration cap, bitwise."""
    pn, on = lattice_pair(23, 50000, 1)
    F = batch_F(2)
    relax = P.RelaxConfig(max_iterations=300)
    br, st, shapes = run([pn], [0, 0], F, tangent=False, relax=relax)
    assert shapes[0]["cluster"] == 16
    resp, status, ost = oracle_batch([on], [0, 0], F, tangent=False,
                                     relax=O.RelaxConfig(max_iterations=300))
    assert list(status) == [6, 6] and br.failed == [0, 1]
    check_states(st, ost)


def test_cluster_lattice_converged(oracle_lib):
    """A mid-size lattice relaxed to convergence, stress and tangent bitwise."""
    pn, on = lattice_pair(12, 6000, 5)
    F = batch_F(2)
    br, st, shapes = run([pn], [0, 0], F, tangent=True)
    assert shapes[0]["cluster"] >= 2
    resp, status, ost = oracle_batch([on], [0, 0], F, tangent=True)
    check_records(br, resp, status, tangent=True)
    check_states(st, ost)


def config3_pair(p):
    from paper_2306_09427_b200 import synth
    pn = synth.config3_network(p)
    on = O.Network(pn.coords, pn.fiber_nodes[:, 0], pn.fiber_nodes[:, 1], pn.fiber_area,
                   pn.fiber_modulus, pn.box_half)
    return pn, on, synth.batch_F(p + 1)[p:p + 1]


@pytest.mark.parametrize("p,force", [(27, None), (1439, 2), (280, 2)])
def test_config3_regressions(oracle_lib, p, force):
    """Config-3 points that once differed: p=27 fills every fiber slot of the (512, 4, 1)
    shape (its schedule has conflicting fiber groups), p=1439/280 on a mirror-mode 2-CTA
    cluster (real fibers whose tail is a halo node)."""
    pn, on, F = config3_pair(p)
    br, st, shapes = run([pn], [0], F, tangent=False, force_cluster=force)
    if force:
        assert shapes[0]["cluster"] == force
    resp, status, ost = oracle_batch([on], [0], F, tangent=False)
    check_records(br, resp, status, tangent=False)
    check_states(st, ost, points=[p_ for p_ in range(1) if not status[p_]])


@pytest.mark.parametrize("kernel", ["edge", "node"])
def test_multiclass_head_launches_tangent(oracle_lib, monkeypatch, kernel):
    """Four config-3 networks in several kernel classes (edge kernel: two resident shapes, a
    large resident shape, a 2-CTA cluster; node kernel: two node shapes and a 2-CTA cluster)
    with the tangent: the multi-class path launches a head and a body grid per class on one
    ticket queue, and probes follow base completion across both launches -- records and
    states bitwise."""
    monkeypatch.setenv("FIBRA_KERNEL", kernel)
    pairs = [config3_pair(p) for p in (1439, 27, 0, 5)]
    pn, on = [q[0] for q in pairs], [q[1] for q in pairs]
    eop = [0, 1, 2, 3, 3, 2, 1, 0]
    F = batch_F(len(eop))
    relax = P.RelaxConfig(tolerance=1e-4)
    br, st, shapes = run(pn, eop, F, tangent=True, relax=relax)
    kinds = {(s["cluster"], s["threads"], s["fibers_per_thread"]) for s in shapes}
    assert len(kinds) == (4 if kernel == "edge" else 3), shapes
    resp, status, ost = oracle_batch(on, eop, F, tangent=True,
                                     relax=O.RelaxConfig(tolerance=1e-4))
    assert not any(status), status
    assert sum(int(r["relax_iterations"]) for r in resp) > 5000
    check_records(br, resp, status, tangent=True)
    check_states(st, ost, points=[p for p in range(len(eop)) if not status[p]])
