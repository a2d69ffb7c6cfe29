"""GPU parity on the inputs the other suites do not reach (bitwise against the oracle):

* per-fibre area and modulus (the non-uniform-EA kernel instances: each fibre's EA in a
  register instead of one scalar), on the resident and the cluster kernels;
* the reference's `segments` generator (netgen.cpp:162-214): node-heavy networks with
  dangling fibres, which select the (512, 6, 2) and (768, 7, 2) resident shapes and, at
  2.5k fibres, a cluster -- checked through their full state after an iteration cap.
"""
import numpy as np
import pytest

import oracle as O
import paper_2306_09427_b200 as P
from _pairs import batch_F, knn, oracle_batch, same_bits

pytestmark = pytest.mark.gpu

STATE_KEYS = ("u", "v", "a", "f_int", "f_damp", "mass", "inv_mass", "t", "iters", "converged")


def solve(pn, on, F, relax=None, tangent=False):
    lib = P.RveLibrary([pn])
    n = len(F)
    st, assign = P.init_batch(np.zeros(n, np.int32), lib, 0)
    db = P.DeviceBatch(lib, assign)
    shape = db.entry_kernel(0)
    db.close()
    br = P.batch_response(lib, assign, st, P.FiberLaw(), F, relax or P.RelaxConfig(),
                          P.StiffnessConfig(), want_tangent=tangent)
    orelax = O.RelaxConfig(max_iterations=relax.max_iterations) if relax else None
    resp, status, ost = oracle_batch([on], [0] * n, F, tangent=tangent, relax=orelax)
    return br, st, resp, status, ost, shape


def check(br, st, resp, status, ost, tangent):
    assert br.failed == list(np.nonzero(status)[0])
    for p, r in enumerate(br.records):
        if status[p]:
            continue
        assert r["base_report"]["iterations"] == resp[p]["base_report"]["iterations"]
        assert same_bits(r["sigma"], resp[p]["sigma"])
        if tangent:
            assert same_bits(r["spatial_c"].reshape(6, 6), resp[p]["spatial_c"])
    for k in STATE_KEYS:
        assert same_bits(getattr(st, k), ost.arrays[k]), k


def with_random_ea(pn, seed):
    rng = np.random.default_rng(seed)
    m = len(pn.fiber_nodes)
    area = rng.uniform(0.5, 1.5, m)
    modulus = rng.uniform(0.8, 1.2, m)
    net = P.FiberNetwork.from_arrays(pn.coords, pn.fiber_nodes, area, modulus, pn.box_half)
    onet = O.Network(net.coords, net.fiber_nodes[:, 0], net.fiber_nodes[:, 1], net.fiber_area,
                     net.fiber_modulus, net.box_half)
    return net, onet


@pytest.mark.parametrize("size,force", [((375, 1000, 1), None), ((712, 1900, 7), "2")])
def test_nonuniform_ea_bitwise(oracle_lib, size, force, monkeypatch):
    if force:  # the cluster kernel's non-uniform-EA instances
        monkeypatch.setenv("FIBRA_FORCE_CLUSTER", force)
    pn, _ = knn(*size)
    net, onet = with_random_ea(pn, 17)
    assert not np.all(net.fiber_area == net.fiber_area[0])
    br, st, resp, status, ost, shape = solve(net, onet, batch_F(3), tangent=True)
    assert shape["cluster"] == (2 if force else 1)
    check(br, st, resp, status, ost, tangent=True)


def test_large_resident_shapes_bitwise(oracle_lib):
    """1.9k-fibre knn RVEs run on one CTA of a large resident shape (g*d record offsets in
    8-byte units), stress and tangent bitwise."""
    pn, on = knn(712, 1900, 7)
    br, st, resp, status, ost, shape = solve(pn, on, batch_F(3), tangent=True)
    assert shape["cluster"] == 1 and shape["fibers_per_thread"] >= 4
    check(br, st, resp, status, ost, tangent=True)


@pytest.mark.parametrize("fibers,seed,cluster", [(300, 1, 1), (1000, 2, 1), (2500, 3, 4)])
def test_segments_networks_capped(oracle_lib, fibers, seed, cluster):
    pn = P.generate_network(P.NetGenSpec(style="segments", fibers=fibers), seed)
    on = O.Network(pn.coords, pn.fiber_nodes[:, 0], pn.fiber_nodes[:, 1], pn.fiber_area,
                   pn.fiber_modulus, pn.box_half)
    br, st, resp, status, ost, shape = solve(pn, on, batch_F(2),
                                             relax=P.RelaxConfig(max_iterations=3000))
    assert shape["cluster"] == cluster
    check(br, st, resp, status, ost, tangent=False)
