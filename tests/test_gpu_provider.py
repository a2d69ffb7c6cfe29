"""NetworkBatchProvider on the GPU (reference batch.cpp:270-302).

Two consecutive `respond` calls (the second warm-started from the device-resident states,
as in a macro Newton loop, macrofem.cpp:347) and `orientation` (orientation_p2,
network.cpp:398-415) of every point, against the oracle running the same sequence on the
same PackedStates -- bitwise.  The library mixes a resident-kernel entry and a cluster
entry.
"""
import numpy as np
import pytest

import oracle as O
import paper_2306_09427_b200 as P
from _pairs import batch_F, knn, same_bits

pytestmark = pytest.mark.gpu


def test_provider_warm_calls_and_orientation(oracle_lib):
    small, osmall = knn(20, 56, 31)
    big = P.generate_lattice_network(12, 6000, 5)  # a cluster entry (beyond the resident shapes)
    obig = O.Network(big.coords, big.fiber_nodes[:, 0], big.fiber_nodes[:, 1], big.fiber_area,
                     big.fiber_modulus, big.box_half)
    lib = P.RveLibrary([small, big])
    n = 6
    prov = P.NetworkBatchProvider(np.zeros(n, np.int32), lib, seed=3)
    eop = prov.assignment.entry_of_point
    assert set(eop.tolist()) == {0, 1}
    onets = [osmall, obig]
    ost = O.PackedStates.fresh(onets, eop)
    F1 = batch_F(n)
    F2 = F1.copy()
    F2[:, 0, 0] += 0.004  # the next macro iterate
    for F in (F1, F2):
        res = prov.respond(F)
        resp, status = O.batch_response(onets, eop, ost, F, want_tangent=True, n_threads=8)
        assert res.failed_points == list(np.nonzero(status)[0])
        assert res.solves_per_point == 7
        assert res.microscale_iterations == sum(int(r["relax_iterations"]) for r in resp)
        for p in range(n):
            assert same_bits(res.responses[p].sigma, resp[p]["sigma"]), p
            assert same_bits(res.responses[p].spatial_c, resp[p]["spatial_c"]), p
    st = prov.states()
    for k in ("u", "v", "f_int", "t", "iters", "converged"):
        assert same_bits(getattr(st, k), ost.arrays[k]), k
    off = np.asarray(st.offsets)
    for d in ([1.0, 0.0, 0.0], [0.0, 0.6, 0.8]):
        for p in range(n):
            a = prov.orientation(p, d)
            b = O.orientation_p2(onets[eop[p]], ost.arrays["u"][off[p]:off[p + 1]], d)
            assert np.float64(a).view(np.uint64) == np.float64(b).view(np.uint64), (p, d)
    assert prov.orientation(n, [1, 0, 0]) is None
