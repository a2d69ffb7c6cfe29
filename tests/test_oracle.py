"""CPU: the oracle restatement (oracle/fibra_oracle.c) pinned to the reference.

* against tests/golden/reference_fixtures.json (made by the reference's own compiled TUs,
  tests/golden/make_golden.py) -- runs everywhere, including the GPU box;
* against oracle/_ref live, bit for bit, where the reference build is present;
* against the closed forms / hand fixtures of the reference's unit tests
  (proj/tests/test_network.cpp, test_relax.cpp, test_stiffness.cpp, test_tensor.cpp).
"""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle as O
import paper_2306_09427_b200 as P
from paper_2306_09427_b200.synth import batch_F

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_fixtures.json")))


def h64(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def onet_from_spec(style, spec, seed):
    pn = P.generate_network(P.NetGenSpec(style=style, **spec), seed)
    return O.Network(pn.coords, pn.fiber_nodes[:, 0], pn.fiber_nodes[:, 1], pn.fiber_area,
                     pn.fiber_modulus)


@pytest.mark.parametrize("g", GOLD["generator"], ids=lambda g: f"{g['style']}-{g['seed']}")
def test_network_layout_matches_reference_fixture(oracle_lib, g):
    on = onet_from_spec(g["style"], {k: (tuple(v) if isinstance(v, list) else v)
                                     for k, v in g["spec"].items()}, g["seed"])
    assert (on.n_nodes, on.n_fibers, on.n_free) == (g["n_nodes"], g["n_fibers"], g["n_free"])
    assert h64(on.coords) == g["coords_sha256"]
    assert h64(np.stack([on.fib_a, on.fib_b])) == g["fibers_sha256"]
    assert h64(on.packed_of_dof) == g["packed_of_dof_sha256"]
    assert h64(on.fiber_dofs) == g["fiber_dofs_sha256"]
    assert h64(on.node_lump) == g["node_lump_sha256"]
    assert h64(on.rest_length) == g["rest_length_sha256"]


@pytest.mark.parametrize("r", GOLD["relax"], ids=lambda r: f"net{r['net']}-{r['F_diag'][0]}")
def test_relax_matches_reference_fixture(oracle_lib, r):
    style, spec, seed = (GOLD["generator"][r["net"]][k] for k in ("style", "spec", "seed"))
    on = onet_from_spec(style, {k: (tuple(v) if isinstance(v, list) else v)
                                for k, v in spec.items()}, seed)
    F = np.diag(r["F_diag"])
    st, rep = O.relax_solve(on, F)
    assert rep["iterations"] == r["iterations"] and rep["converged"] == r["converged"]
    for k in ("residual", "eps_eff", "kinetic_fraction", "dt"):
        assert float(rep[k]).hex() == r[k], k
    assert float(st.t[0]).hex() == r["t"]
    assert h64(st.u) == r["u_sha256"] and h64(st.v) == r["v_sha256"]
    assert h64(st.f_int) == r["f_int_sha256"]
    if rep["converged"]:
        sig, asym = O.homogenized_stress(on, st, F)
        assert [float(x).hex() for x in sig] == r["sigma"] and float(asym).hex() == r["asym"]


def test_batch_F_recipe_matches_reference_rng():
    assert h64(batch_F(16)) == GOLD["batch_F"]["sha256"]


# ---------------------------------------------------------------- live, bitwise vs _ref
ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built here")


@ref
@pytest.mark.parametrize("seed,F", [(31, [1.06, 1.0, 0.97]), (11, [1.04, 0.99, 1.01]),
                                     (41, [1.25, 1.0, 1.0]), (7, [0.96, 1.03, 1.0])])
def test_relax_bitwise_vs_reference_live(oracle_lib, seed, F):
    rn = O.ref_generate("knn", nodes=20, fibers=56, neighbors=10, seed=seed)
    on = O.network_from_ref(rn)
    for law in (O.Law(), O.Law(kind=0, buckling_off=True), O.Law(kind=1, nonlinearity=4.0)):
        s1, r1 = O.relax_solve(on, np.diag(F), law=law)
        s2, r2 = O.ref_relax_solve(rn, np.diag(F), law=law)
        assert r1 == r2
        for k in ("u", "v", "a", "f_int", "f_damp", "mass", "inv_mass", "t", "iters"):
            assert np.array_equal(getattr(s1, k).view(np.uint8), getattr(s2, k).view(np.uint8)), k


@ref
def test_relax_warm_and_capped_vs_reference_live(oracle_lib):
    rn = O.ref_generate("knn", nodes=16, fibers=44, neighbors=10, seed=21)
    on = O.network_from_ref(rn)
    F = np.diag([1.03, 1.0, 0.99])
    s1, _ = O.relax_solve(on, F)
    s2, _ = O.ref_relax_solve(rn, F)
    F2 = np.array([[1.035, 0.01, 0], [0, 0.995, 0], [0, 0, 1.0]])
    cfg = O.RelaxConfig(max_iterations=37, damping=1.5, dt_safety=0.7)
    a, ra = O.relax_solve(on, F2, cfg=cfg, state=s1, warm_reuse=True)
    b, rb = O.ref_relax_solve(rn, F2, cfg=cfg, state=s2, warm_reuse=True)
    assert ra == rb and not ra["converged"] and ra["iterations"] == 37
    for k in ("u", "v", "a", "f_int", "t", "iters"):
        assert np.array_equal(getattr(a, k).view(np.uint8), getattr(b, k).view(np.uint8)), k


@ref
def test_orientation_p2_bitwise_vs_reference_live(oracle_lib):
    """orientation_p2 (network.cpp:398-415) on a relaxed state and on the reference state."""
    rn = O.ref_generate("knn", nodes=40, fibers=110, neighbors=10, seed=5)
    on = O.network_from_ref(rn)
    s, _ = O.ref_relax_solve(rn, np.diag([1.2, 0.95, 1.0]))
    for d in ([1.0, 0.0, 0.0], [0.0, 0.6, 0.8], [0.3, -0.4, 0.8660254037844386]):
        for u in (s.u, np.zeros_like(s.u)):
            a = O.orientation_p2(on, u, d)
            b = O.ref_orientation_p2(rn, u, d)
            assert np.float64(a).view(np.uint64) == np.float64(b).view(np.uint64)
    # stretching along x aligns fibres with x: P2 grows
    assert O.orientation_p2(on, s.u, [1, 0, 0]) > O.orientation_p2(on, np.zeros_like(s.u), [1, 0, 0])


@ref
def test_internal_forces_bitwise_vs_reference_live(oracle_lib):
    rn = O.ref_generate("knn", nodes=60, fibers=200, neighbors=8, seed=3)
    on = O.network_from_ref(rn)
    rng = np.random.default_rng(0)
    for law in (O.Law(), O.Law(kind=1, nonlinearity=2.0), O.Law(buckling_off=True)):
        u = rng.normal(scale=0.01, size=on.n_dof)
        f1 = O.internal_forces(on, u, law)
        f2 = np.zeros(on.n_dof)
        O.ref().ref_internal_forces(rn.h, law.kind, law.ea_scale, law.nonlinearity,
                                    int(law.buckling_off), O._ptr(u, O._dp), O._ptr(f2, O._dp))
        assert np.array_equal(f1.view(np.uint64), f2.view(np.uint64))


# -------------------------------------------------- reference unit-test closed forms
def single_fiber():  # oracles.cpp:155-159
    return O.Network([[-0.5, 0, 0], [0.5, 0, 0]], [0], [1])


def two_segment_chain():  # oracles.cpp:161-174
    mid, ea1, ea2 = -0.1, 2.0, 1.0
    net = O.Network([[-0.5, 0, 0], [mid, 0, 0], [0.5, 0, 0]], [0, 1], [1, 2], [1.0, 1.0],
                    [ea1, ea2])
    l1, l2 = mid + 0.5, 0.5 - mid

    def interior_x(lam):
        k1, k2 = ea1 / l1, ea2 / l2
        return (0.5 * lam * (k2 - k1) + ea1 - ea2) / (k1 + k2)
    return net, interior_x, ea1, mid


def test_single_fiber_axial_force(oracle_lib):  # test_network.cpp:164-176
    net = single_fiber()
    lam = 1.25
    st = O.State(net.n_dof, net.n_free)
    O.lib().or_apply_affine_bc(O.C.byref(net.c), O._F(np.diag([lam, 1, 1])).ctypes.data_as(O._dp), st.c())
    f = O.internal_forces(net, st.u)
    fr = f[net.packed_of_dof[3 * 1]]
    assert abs(fr - (lam - 1)) <= 1e-14 * (lam - 1)
    assert st.u[net.packed_of_dof[3]] == 0.125  # affine BC value exact


def test_homogenized_stress_closed_form(oracle_lib):  # test_network.cpp:285-301
    net = single_fiber()
    lam = 1.2
    st, rep = O.relax_solve(net, np.diag([lam, 1, 1]))
    assert rep["converged"] and rep["iterations"] == 0  # no free dofs
    sig, asym = O.homogenized_stress(net, st, np.diag([lam, 1, 1]))
    want = (lam - 1.0) * lam / (lam * 1.0)
    assert abs(sig[0] - want) <= 1e-12 * want and abs(sig[1]) <= 1e-15 and asym <= 1e-12


def test_chain_closed_form_and_reactions(oracle_lib):  # test_relax.cpp:71-88
    net, interior_x, ea1, mid = two_segment_chain()
    lam = 1.3
    st, rep = O.relax_solve(net, np.diag([lam, 1, 1]), cfg=O.RelaxConfig(tolerance=1e-10))
    assert rep["converged"]
    x_mid = mid + st.u[net.packed_of_dof[3 * 1]]
    assert abs(x_mid - interior_x(lam)) <= 1e-8 * abs(interior_x(lam))
    n1 = ea1 * ((x_mid + lam / 2) / (mid + 0.5) - 1.0)
    assert abs(-st.f_int[net.packed_of_dof[0]] - n1) <= 1e-8 * max(1.0, n1)


def test_identity_and_cap(oracle_lib):  # test_relax.cpp:51-69
    net, *_ = two_segment_chain()
    st, rep = O.relax_solve(net, np.eye(3))
    assert rep["converged"] and rep["iterations"] == 0 and rep["residual"] == 0.0
    st, rep = O.relax_solve(net, np.diag([1.3, 1, 1]), cfg=O.RelaxConfig(max_iterations=2))
    assert not rep["converged"] and rep["iterations"] == 2 and st.converged[0] == 0


def test_relax_properties(oracle_lib):  # test_relax.cpp:140-185
    on = onet_from_spec("knn", dict(nodes=20, fibers=56, neighbors=10), 31)
    F = np.diag([1.06, 1.0, 0.97])
    st, rep = O.relax_solve(on, F)
    f = O.internal_forces(on, st.u)
    res = np.sqrt(O.norm2_sq(f[:on.n_free]))
    assert res <= rep["eps_eff"] and res == rep["residual"]      # certificate, bitwise
    assert np.all(st.v[on.n_free:] == 0) and np.all(st.a[on.n_free:] == 0)
    st2, rep2 = O.relax_solve(on, F, state=st, warm_reuse=True)  # warm start
    assert rep2["converged"] and rep2["iterations"] <= 2
    s3, r3 = O.relax_solve(on, F)                                # determinism
    assert r3 == rep and np.array_equal(s3.u, st.u)


def test_divergence_named(oracle_lib):  # test_relax.cpp:231-239
    net, *_ = two_segment_chain()
    with pytest.raises(O.OracleError) as e:
        O.relax_solve(net, np.diag([1.2, 1, 1]), cfg=O.RelaxConfig(damping=1e9, max_iterations=100000))
    assert e.value.code == 5  # OR_DIVERGED


def test_polar_properties(oracle_lib):  # test_tensor.cpp:59-112 (tolerance-pinned Eigen step)
    rng = np.random.default_rng(3)
    for _ in range(200):
        F = np.eye(3) + rng.uniform(-0.3, 0.3, (3, 3))
        if np.linalg.det(F) < 0.2:
            continue
        R, U = O.polar_decompose(F)
        Uf = np.array([[U[0], U[5], U[4]], [U[5], U[1], U[3]], [U[4], U[3], U[2]]])
        assert np.linalg.norm(F - R @ Uf) <= 1e-10 * np.linalg.norm(F)
        assert np.linalg.norm(R.T @ R - np.eye(3)) <= 1e-12
        assert np.all(np.linalg.eigvalsh(Uf) > 0)
    R, U = O.polar_decompose(np.diag([1.05, 1.0, 1.0]))  # diagonal F: U exact
    assert list(U) == [1.05, 1.0, 1.0, 0.0, 0.0, 0.0]
    with pytest.raises(O.OracleError):
        O.polar_decompose(np.diag([-1.0, 1, 1]))


def test_eigen_sym3_restatement(oracle_lib):
    """Eigen 3.4.0 SelfAdjointEigenSolver<Matrix3d> restatement (fibra_oracle.c): agrees
    with LAPACK to rounding, ascending order, orthonormal columns; a diagonal input deflates
    without a QR step, so eigenvalues are the diagonal bits exactly (sorted) and Q is a
    permutation."""
    rng = np.random.default_rng(11)
    for t in range(2000):
        F = np.eye(3) + rng.uniform(-0.3, 0.3, (3, 3)) * 10.0 ** rng.uniform(-8, 0)
        C = F.T @ F
        lam, Q = O.eigen_sym3(C)
        assert np.all(np.diff(lam) >= 0)
        assert np.max(np.abs(lam - np.linalg.eigvalsh(C))) <= 1e-14 * np.max(np.abs(lam))
        assert np.linalg.norm(C @ Q - Q * lam) <= 1e-14 * np.linalg.norm(C)
        assert np.linalg.norm(Q.T @ Q - np.eye(3)) <= 1e-14
    lam, Q = O.eigen_sym3(np.diag([3.0, 1.0, 2.0]))
    assert list(lam) == [1.0, 2.0, 3.0]
    assert sorted(map(tuple, np.abs(Q))) == sorted(map(tuple, np.eye(3)))


def _substitute_pk2(U6, mu=1.3, lam=0.8):  # batch.cpp:199-214 (closed-form material)
    U = np.array([[U6[0], U6[5], U6[4]], [U6[5], U6[1], U6[3]], [U6[4], U6[3], U6[2]]])
    C = U @ U
    Ci = np.linalg.inv(C)
    S = mu * (np.eye(3) - Ci) + lam * np.log(np.linalg.det(U)) * Ci
    return np.array([S[0, 0], S[1, 1], S[2, 2], S[1, 2], S[0, 2], S[0, 1]])


def _substitute_tangent(U6, mu=1.3, lam=0.8):  # batch.cpp:216-236
    U = np.array([[U6[0], U6[5], U6[4]], [U6[5], U6[1], U6[3]], [U6[4], U6[3], U6[2]]])
    Ci = np.linalg.inv(U @ U)
    I, J = [0, 1, 2, 1, 0, 0], [0, 1, 2, 2, 2, 1]
    vci = np.array([Ci[I[q], J[q]] * (1 if q < 3 else np.sqrt(2)) for q in range(6)])
    g = 2.0 * (mu - lam * np.log(np.linalg.det(U)))
    A = np.zeros((6, 6))
    for q in range(6):
        for r in range(6):
            wq = 1 if q < 3 else np.sqrt(2)
            wr = 1 if r < 3 else np.sqrt(2)
            sym = 0.5 * (Ci[I[q], I[r]] * Ci[J[q], J[r]] + Ci[I[q], J[r]] * Ci[J[q], I[r]])
            A[q, r] = lam * vci[q] * vci[r] + g * wq * wr * sym
    return A


def test_probing_pipeline_recovers_analytic_tangent(oracle_lib):  # test_stiffness.cpp:113-126
    L = O.lib()
    rng = np.random.default_rng(3)
    for it in range(6):
        if it == 0:
            U = np.array([1.0, 1, 1, 0, 0, 0])
        else:
            Q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
            Uf = Q @ np.diag(rng.uniform(0.6, 1.6, 3)) @ Q.T
            U = np.array([Uf[0, 0], Uf[1, 1], Uf[2, 2], Uf[1, 2], Uf[0, 2], Uf[0, 1]])
        h = 1e-7 * np.sqrt(U[0] ** 2 + U[1] ** 2 + U[2] ** 2 + 2 * (U[3] ** 2 + U[4] ** 2 + U[5] ** 2))
        base = _substitute_pk2(U)
        probes = np.zeros(36)
        for q in range(6):
            d = np.zeros(6)
            L.or_probing_direction.argtypes = [O.C.c_int, O._dp]
            L.or_probing_direction(q, O._ptr(d, O._dp))
            probes[6 * q:6 * q + 6] = _substitute_pk2(U + d * h)
        A = np.zeros(36)
        rc = L.or_material_stiffness_from_probes(O._ptr(U, O._dp), O._ptr(base, O._dp),
                                                 O._ptr(probes, O._dp), h, O._ptr(A, O._dp))
        assert rc == 0
        A_ref = _substitute_tangent(U)
        assert np.linalg.norm(A.reshape(6, 6) - A_ref) <= 1e-6 * np.linalg.norm(A_ref)


def _condensed_reference_tangent(on):  # test_stiffness.cpp:52-106 restated with numpy
    nd, nf = on.n_dof, on.n_free
    K = np.zeros((nd, nd))
    ref = on.packed_ref
    for f in range(on.n_fibers):
        p = on.fiber_dofs[6 * f:6 * f + 6]
        l0 = on.rest_length[f]
        d = (ref[p[3:]] - ref[p[:3]]) / l0
        ke = np.outer(d, d) * (on.area[f] * on.modulus[f] / l0)
        K[np.ix_(p[:3], p[:3])] += ke
        K[np.ix_(p[3:], p[3:])] += ke
        K[np.ix_(p[:3], p[3:])] -= ke
        K[np.ix_(p[3:], p[:3])] -= ke
    dof_of_packed = np.argsort(on.packed_of_dof)
    C = np.zeros((6, 6))
    I, J = [0, 1, 2, 1, 0, 0], [0, 1, 2, 2, 2, 1]
    for q in range(6):
        eps = np.zeros((3, 3))
        w = 1.0 if q < 3 else 1 / np.sqrt(2)
        eps[I[q], J[q]] = eps[J[q], I[q]] = w
        ub = np.array([eps[dof % 3] @ on.coords[dof // 3] for dof in dof_of_packed[nf:]])
        uf = np.linalg.solve(K[:nf, :nf], -(K[:nf, nf:] @ ub))
        rb = K[nf:, :nf] @ uf + K[nf:, nf:] @ ub
        s = np.zeros((3, 3))
        for i, dof in enumerate(dof_of_packed[nf:]):
            s[dof % 3] += rb[i] * on.coords[dof // 3]
        raw = s / (8 * on.box_half ** 3)
        sym = 0.5 * (raw + raw.T)
        C[:, q] = [sym[0, 0], sym[1, 1], sym[2, 2], np.sqrt(2) * sym[1, 2], np.sqrt(2) * sym[0, 2],
                   np.sqrt(2) * sym[0, 1]]
    return C


def test_network_material_stiffness(oracle_lib):  # test_stiffness.cpp:183-214
    on = onet_from_spec("knn", dict(nodes=20, fibers=56, neighbors=10), 71)
    tight = O.RelaxConfig(tolerance=1e-10, max_iterations=2000000)
    loose = O.RelaxConfig(tolerance=1e-8, max_iterations=2000000)
    F = np.diag([1.05, 1.0, 0.99])
    resp, _ = O.constitutive_response(on, F, relax_cfg=tight)
    assert resp["solves"] == 7 and resp["failed_probe"] == -1
    C = np.zeros(36)
    A = np.ascontiguousarray(resp["material_a"]).reshape(36)
    O.lib().or_push_forward_stiffness(O._ptr(A, O._dp), O._ptr(O._F(F), O._dp), O._ptr(C, O._dp))
    assert np.array_equal(C.reshape(6, 6), resp["spatial_c"])
    r0, _ = O.constitutive_response(on, np.eye(3), relax_cfg=loose)
    assert np.linalg.norm(r0["spatial_c"] - r0["material_a"]) <= 1e-12 * np.linalg.norm(r0["material_a"])
    assert np.linalg.norm(r0["sigma"]) <= 1e-10 and np.linalg.norm(r0["material_a"]) > 0.01
    want = _condensed_reference_tangent(on)
    assert np.linalg.norm(r0["material_a"] - want) <= 1e-3 * np.linalg.norm(want)


def test_batch_threads_bitwise_equal_sequential(oracle_lib):  # test_batch.cpp:134-178
    nets = [onet_from_spec("knn", dict(nodes=14, fibers=38, neighbors=9), 101),
            onet_from_spec("knn", dict(nodes=12, fibers=32, neighbors=9), 102)]
    eop = [1, 0, 0, 1, 1, 0, 1, 0]
    F = batch_F(8)
    st1 = O.PackedStates.fresh(nets, eop)
    r1, s1 = O.batch_response(nets, eop, st1, F, n_threads=1)
    st4 = O.PackedStates.fresh(nets, eop)
    r4, s4 = O.batch_response(nets, eop, st4, F, n_threads=4)
    assert not s1.any() and np.array_equal(s1, s4)
    for a, b in zip(r1, r4):
        assert np.array_equal(a["sigma"], b["sigma"]) and np.array_equal(a["spatial_c"], b["spatial_c"])
    for k in ("u", "v", "f_int"):
        assert np.array_equal(st1.arrays[k], st4.arrays[k])


def test_config2_fixture_pins_polar_and_solves(oracle_lib):
    """tests/golden/config2_full.json (reference build, make_golden_batches.py): the oracle's
    Eigen 3.4.0 polar restatement reproduces the fixture's U bits for all 1,024 config-2 F,
    and the oracle's relax reproduces the reference's iterations and sigma on the cheapest
    points (the GPU suite checks all of them)."""
    import json
    import os
    from oracle import workload as W
    path = os.path.join(os.path.dirname(__file__), "golden", "config2_full.json")
    with open(path) as fh:
        pts = json.load(fh)["points"]
    F = W.batch_F(len(pts))
    for q in pts:
        R, U = O.polar_decompose(F[q["p"]])
        assert list(U.view(np.uint64)) == [np.float64(float.fromhex(x)).view(np.uint64)
                                           for x in q["U"]], q["p"]
    cheap = sorted((q for q in pts if q["status"] == 0), key=lambda q: q["base_iterations"])[:4]
    import paper_2306_09427_b200 as P
    from paper_2306_09427_b200 import synth
    pn = P.generate_network(synth.config1_spec(), 1)
    on = O.Network(pn.coords, pn.fiber_nodes[:, 0], pn.fiber_nodes[:, 1], pn.fiber_area,
                   pn.fiber_modulus, pn.box_half)
    ids = [q["p"] for q in cheap]
    st = O.PackedStates.fresh([on], [0] * len(ids))
    resp, status = O.batch_response([on], [0] * len(ids), st, F[ids], want_tangent=False)
    for i, q in enumerate(cheap):
        assert status[i] == 0
        assert resp[i]["base_report"]["iterations"] == q["base_iterations"]
        assert [float(x).hex() for x in resp[i]["sigma"]] == q["sigma"]
