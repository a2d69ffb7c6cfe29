"""Macro assembly oracle and host logic (CPU).

The oracle's assemble (oracle/fibra_oracle.c or_assemble, restating macrofem.cpp:104-187)
is pinned to the reference's own known answers for this path -- tests/test_macrofem.cpp:44-83
("b_matrix on the canonical tet") and :109-177 ("assembly": zero stress -> zero residual,
single-tet hand integration, stiffness = central FD of the residual to 1e-6, element order
permutation) -- plus the error order of macrofem.cpp:118-132.  Eigen is absent here, so its
3x3 determinant/inverse and setFromTriplets folding are restated.
"""
import numpy as np
import pytest

import oracle as O
from paper_2306_09427_b200.assembly import (DirichletBc, build_numbering, make_box_mesh)


def element_F(mesh, e):
    """deformation_of_element (test_macrofem.cpp:18-28 / macrofem.cpp:89-100)."""
    g0, _ = O.tet_geom(mesh.ref_coords.ravel(), mesh.tets[e])
    x = mesh.coords[mesh.tets[e]]
    return x.T @ g0


def neo_hooke(F, mu, lam):
    """Compressible neo-Hookean Cauchy stress and spatial tangent (the closed form of
    substitute_response, batch.cpp:233-249): c = lam/J m m^T + 2 (mu - lam ln J)/J I6."""
    J = np.linalg.det(F)
    b = F @ F.T
    s = (mu * (b - np.eye(3)) + lam * np.log(J) * np.eye(3)) / J
    sig = np.array([s[0, 0], s[1, 1], s[2, 2], s[1, 2], s[0, 2], s[0, 1]])
    m = np.array([1.0, 1, 1, 0, 0, 0])
    c = lam / J * np.outer(m, m) + 2 * (mu - lam * np.log(J)) / J * np.eye(6)
    return sig, c


def substitute(mesh, mu=1.2, lam=0.9):
    sig, cm = zip(*(neo_hooke(element_F(mesh, e), mu, lam) for e in range(mesh.n_elements)))
    return np.array(sig), np.array(cm)


def dense(res, cp, ri, va):
    n = len(res)
    K = np.zeros((n, n))
    for c in range(n):
        K[ri[cp[c]:cp[c + 1]], c] = va[cp[c]:cp[c + 1]]
    return K


def test_canonical_tet(oracle_lib):  # test_macrofem.cpp:44-57
    coords = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)
    g, v = O.tet_geom(coords.ravel(), [0, 1, 2, 3])
    assert v == pytest.approx(1 / 6)
    assert np.array_equal(g, [[-1, -1, -1], [1, 0, 0], [0, 1, 0], [0, 0, 1]])
    with pytest.raises(O.OracleError) as ei:  # test_macrofem.cpp:78-82 (inverted)
        O.tet_geom(coords.ravel(), [0, 2, 1, 3])
    assert ei.value.code == 2


def test_box_mesh_and_numbering():
    mesh = make_box_mesh(2, 3, 1, 1.0, 1.5, 0.5)
    assert mesh.n_nodes == 3 * 4 * 2 and mesh.n_elements == 6 * 6
    for e in range(mesh.n_elements):
        _, v = O.tet_geom(mesh.ref_coords.ravel(), mesh.tets[e])
        assert v > 0
    assert np.sum([O.tet_geom(mesh.ref_coords.ravel(), t)[1] for t in mesh.tets]) == \
        pytest.approx(1.0 * 1.5 * 0.5)
    num = build_numbering(mesh, [DirichletBc("xmin", affine=np.eye(3)),
                                 DirichletBc("zmax", value=(None, None, 0.1))])
    xmin, zmax = mesh.node_sets["xmin"], mesh.node_sets["zmax"]
    assert num.constrained[3 * xmin].all() and num.constrained[3 * xmin + 2].all()
    assert num.constrained[3 * zmax + 2].all()
    assert num.n_free == mesh.n_dof - 3 * len(xmin) - len(np.setdiff1d(zmax, xmin))
    free = num.free_of_dof[num.free_of_dof >= 0]
    assert np.array_equal(free, np.arange(num.n_free))


def test_zero_stress_and_hand_integration(oracle_lib):  # test_macrofem.cpp:115-139
    mesh = make_box_mesh(1, 1, 1)
    num = build_numbering(mesh)
    n = mesh.n_elements
    c = np.tile(np.eye(6).ravel(), (n, 1))
    res, cp, ri, va = O.assemble(mesh.tets, mesh.coords.ravel(), np.zeros((n, 6)), c,
                                 num.free_of_dof, num.n_free)
    assert np.linalg.norm(res) == 0.0
    one = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)
    sig = np.array([[2.5, 0, 0, 0, 0, 0]])
    fod = np.arange(12, dtype=np.int32)
    res, cp, ri, va = O.assemble([[0, 1, 2, 3]], one.ravel(), sig, np.zeros((1, 36)), fod, 12)
    g, v = O.tet_geom(one.ravel(), [0, 1, 2, 3])
    for node in range(4):
        assert res[3 * node] == pytest.approx(v * 2.5 * g[node, 0])
        assert res[3 * node + 1] == pytest.approx(0.0)
    assert len(va) == 144 and np.array_equal(cp, np.arange(13) * 12)


def test_stiffness_is_fd_of_residual(oracle_lib):  # test_macrofem.cpp:141-162
    rng = np.random.default_rng(17)
    mesh = make_box_mesh(1, 1, 1)
    num = build_numbering(mesh)
    mesh.coords = mesh.ref_coords + rng.uniform(-0.03, 0.03, mesh.ref_coords.shape)

    def asm(m):
        sig, cm = substitute(m)
        return O.assemble(m.tets, m.coords.ravel(), sig, cm, num.free_of_dof, num.n_free)

    base = asm(mesh)
    K = dense(*base)
    eps, max_rel = 1e-6, 0.0
    for d in range(0, num.n_free, 7):
        mp, mm = make_box_mesh(1, 1, 1), make_box_mesh(1, 1, 1)
        mp.coords, mm.coords = mesh.coords.copy(), mesh.coords.copy()
        mp.coords[d // 3, d % 3] += eps
        mm.coords[d // 3, d % 3] -= eps
        fd = (asm(mp)[0] - asm(mm)[0]) / (2 * eps)
        max_rel = max(max_rel, np.linalg.norm(fd - K[:, d]) / np.linalg.norm(K[:, d]))
    assert max_rel <= 1e-6


def test_element_permutation(oracle_lib):  # test_macrofem.cpp:164-177
    mesh = make_box_mesh(1, 1, 1)
    num = build_numbering(mesh)
    mesh.coords = mesh.ref_coords * 1.02
    sig, cm = substitute(mesh, 1.0, 1.0)
    a = O.assemble(mesh.tets, mesh.coords.ravel(), sig, cm, num.free_of_dof, num.n_free)
    b = O.assemble(mesh.tets[::-1], mesh.coords.ravel(), sig[::-1], cm[::-1], num.free_of_dof,
                   num.n_free)
    assert np.linalg.norm(a[0] - b[0]) <= 1e-12 * max(1.0, np.linalg.norm(a[0]))
    Ka, Kb = dense(*a), dense(*b)
    assert np.linalg.norm(Ka - Kb) <= 1e-12 * np.linalg.norm(Ka)
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


def test_error_order(oracle_lib):  # macrofem.cpp:118-132: first failing element wins
    mesh = make_box_mesh(2, 1, 1)
    num = build_numbering(mesh)
    n = mesh.n_elements
    sig = np.zeros((n, 6))
    cm = np.tile(np.eye(6).ravel(), (n, 1))
    sig[7, 3] = np.nan
    bad = mesh.tets.copy()
    bad[4, 2], bad[4, 3] = bad[4, 3], bad[4, 2]  # inverted element before the NaN
    with pytest.raises(O.OracleError) as ei:
        O.assemble(bad, mesh.coords.ravel(), sig, cm, num.free_of_dof, num.n_free)
    assert ei.value.code == 2 and ei.value.element == 4
    with pytest.raises(O.OracleError) as ei:
        O.assemble(mesh.tets, mesh.coords.ravel(), sig, cm, num.free_of_dof, num.n_free)
    assert ei.value.code == 10 and ei.value.element == 7
    f = np.zeros(num.n_free)
    f[3] = np.inf
    with pytest.raises(O.OracleError) as ei:
        O.assemble(mesh.tets, mesh.coords.ravel(), np.zeros((n, 6)), cm, num.free_of_dof,
                   num.n_free, f)
    assert ei.value.code == 11


def test_assembly_create_rejects_bad_numbering():
    """fibra_cuda_assembly_create validates the DOF numbering before any device work: free
    slots must be 0..n_free-1 in ascending DOF order (build_numbering, macrofem.cpp:22-38),
    else FIBRA_E_ARG (a shared or out-of-order slot would break the CSC pattern)."""
    import ctypes as C
    from paper_2306_09427_b200 import _capi
    L = _capi.load()
    tets = np.array([0, 1, 2, 3], np.int32)
    h = C.c_void_p()
    for fod in ([0, 1, 2, -1, -1, -1, 3, 4, 5, -1, -1, 5],   # slot 5 twice
                [1, 0, 2, -1, -1, -1, 3, 4, 5, -1, -1, -1],  # descending
                [0, 1, 2, -1, -1, -1, 3, 4, 6, -1, -1, -1]):  # gap
        f = np.array(fod, np.int32)
        rc = L.fibra_cuda_assembly_create(0, tets.ctypes.data_as(_capi._ip), 1, 4,
                                          f.ctypes.data_as(_capi._ip), 6, C.byref(h))
        assert rc == 21, fod  # FIBRA_E_ARG
