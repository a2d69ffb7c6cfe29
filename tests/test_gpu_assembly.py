"""Device macro assembly (csrc/assembly.cu) against the oracle, bit for bit.

Reference: fibra::assemble, macrofem.cpp:104-187.  Same inputs to both; the sparsity
pattern, the residual and every stiffness value must match the oracle's restatement of
Eigen's setFromTriplets exactly (uint64 views, so -0.0 vs +0.0 counts).
"""
import numpy as np
import pytest

import oracle as O
import paper_2306_09427_b200 as P
from paper_2306_09427_b200.assembly import (DirichletBc, MacroAssembler, assemble,
                                            build_numbering, make_box_mesh)

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def case(nx, ny, nz, seed, bcs=True):
    rng = np.random.default_rng(seed)
    mesh = make_box_mesh(nx, ny, nz, 1.0, 0.8, 1.3)
    h = min(1.0 / nx, 0.8 / ny, 1.3 / nz)
    mesh.coords = mesh.ref_coords + rng.uniform(-0.08 * h, 0.08 * h, mesh.ref_coords.shape)
    dbc = [DirichletBc("xmin", affine=np.eye(3)), DirichletBc("zmax", value=(None, 0.0, 0.1))]
    num = build_numbering(mesh, dbc if bcs else [])
    n = mesh.n_elements
    sig = rng.standard_normal((n, 6))
    sig[rng.random((n, 6)) < 0.1] = 0.0  # exact zeros: signed-zero paths
    cm = rng.standard_normal((n, 36))
    f_ext = rng.standard_normal(num.n_free)
    return mesh, num, sig, cm, f_ext


def check_equal(asm, ref):
    res, cp, ri, va = ref
    assert np.array_equal(asm.col_ptr, cp) and np.array_equal(asm.row_idx, ri)
    assert np.array_equal(bits(asm.residual), bits(res))
    assert np.array_equal(bits(asm.values), bits(va))


@pytest.mark.parametrize("dims,seed,bcs", [((1, 1, 1), 1, False), ((3, 2, 2), 2, True),
                                           ((12, 10, 9), 3, True)])
def test_assembly_bitwise(oracle_lib, dims, seed, bcs):
    mesh, num, sig, cm, f_ext = case(*dims, seed, bcs)
    ref = O.assemble(mesh.tets, mesh.coords.ravel(), sig, cm, num.free_of_dof, num.n_free, f_ext)
    A = MacroAssembler(mesh, num)
    check_equal(A.assemble(mesh.coords, sig, cm, f_ext), ref)
    # repeated calls on the same plan, no f_ext (= zero vector)
    ref0 = O.assemble(mesh.tets, mesh.coords.ravel(), sig, cm, num.free_of_dof, num.n_free)
    check_equal(A.assemble(mesh.coords, sig, cm), ref0)
    info = A.info()
    assert info["nnz"] == len(ref[3]) and info["n_free"] == num.n_free


def test_assembly_errors(oracle_lib):
    mesh, num, sig, cm, _ = case(3, 2, 2, 5)
    bad = mesh.tets.copy()
    bad[9, 2], bad[9, 3] = bad[9, 3], bad[9, 2]
    sig[20, 1] = np.inf
    mesh_bad = make_box_mesh(3, 2, 2, 1.0, 0.8, 1.3)
    mesh_bad.coords, mesh_bad.tets = mesh.coords, bad
    for m, code, elem, exc in ((mesh_bad, 2, 9, P.KinematicsError), (mesh, 10, 20, P.SolverError)):
        with pytest.raises(O.OracleError) as oe:
            O.assemble(m.tets, m.coords.ravel(), sig, cm, num.free_of_dof, num.n_free)
        assert oe.value.code == code and oe.value.element == elem
        with pytest.raises(exc, match=f"element {elem}"):
            MacroAssembler(m, num).assemble(m.coords, sig, cm)
    sig[20, 1] = 0.0
    f = np.zeros(num.n_free)
    f[5] = np.nan
    with pytest.raises(P.SolverError, match="residual"):
        MacroAssembler(mesh, num).assemble(mesh.coords, sig, cm, f)


def test_assembly_of_solved_responses(oracle_lib):
    """The consumer of batch_response: one RVE point per tet, F from each element's
    deformation, solved on the device, then assembled from the fibra_point_result records
    (host stride path) and from the same records left in HBM (device path)."""
    import torch

    rng = np.random.default_rng(11)
    mesh = make_box_mesh(1, 1, 1)
    mesh.coords = mesh.ref_coords * np.array([1.01, 0.995, 1.0]) + \
        rng.uniform(-0.002, 0.002, mesh.ref_coords.shape)
    num = build_numbering(mesh, [DirichletBc("xmin", affine=np.eye(3))])
    n = mesh.n_elements
    F = np.zeros((n, 3, 3))
    for e in range(n):
        g0, _ = O.tet_geom(mesh.ref_coords.ravel(), mesh.tets[e])
        F[e] = mesh.coords[mesh.tets[e]].T @ g0
    net = P.generate_network(P.NetGenSpec(style="knn", nodes=20, fibers=56, neighbors=10), 31)
    lib = P.RveLibrary([net])
    states, assign = P.init_batch(np.zeros(n, np.int32), lib, 0)
    br = P.batch_response(lib, assign, states, P.FiberLaw(), F.reshape(n, 9), P.RelaxConfig(),
                          P.StiffnessConfig(), device=0)
    assert br.failed == []
    sig = np.array([r.sigma for r in br.responses])
    cm = np.array([r.spatial_c.ravel() for r in br.responses])
    ref = O.assemble(mesh.tets, mesh.coords.ravel(), sig, cm, num.free_of_dof, num.n_free)
    rec = np.ascontiguousarray(br.records)
    stride = rec.dtype.itemsize // 8
    A = MacroAssembler(mesh, num)
    check_equal(A.assemble(mesh.coords, responses=rec, stride=stride), ref)
    # the reference-facing one-shot call with PointResponse objects
    check_equal(assemble(mesh, num, br.responses), ref)
    # device path: records and coords in HBM, outputs in HBM
    dev = torch.device("cuda:0")
    d_rec = torch.from_numpy(rec.view(np.uint8).copy()).to(dev)
    d_x = torch.from_numpy(np.ascontiguousarray(mesh.coords)).to(dev)
    d_res = torch.empty(num.n_free, dtype=torch.float64, device=dev)
    d_val = torch.empty(A.nnz, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    A.assemble_device(d_x.data_ptr(), d_rec.data_ptr(), stride, None, d_res.data_ptr(),
                      d_val.data_ptr())
    A.status()
    assert np.array_equal(bits(d_res.cpu().numpy()), bits(ref[0]))
    assert np.array_equal(bits(d_val.cpu().numpy()), bits(ref[3]))


def test_assembly_nonfinite_tangent(oracle_lib):
    """The reference checks only sigma (macrofem.cpp:122-125); an inf in C propagates into
    K as inf/NaN.  Those elements take the kernel's dense path (the structural-zero skip is
    exact only for finite factors); compare with NaN == NaN (payload bits differ between
    x86 and the GPU) and bitwise everywhere else."""
    mesh, num, sig, cm, f_ext = case(3, 2, 2, 9)
    cm[4, 7] = np.inf
    cm[30, 0] = -np.inf
    cm[31, 13] = np.nan
    sig[12] = 1e300  # C B finite, but products overflow in K
    res, cp, ri, va = O.assemble(mesh.tets, mesh.coords.ravel(), sig, cm, num.free_of_dof,
                                 num.n_free, f_ext)
    asm = MacroAssembler(mesh, num).assemble(mesh.coords, sig, cm, f_ext)
    assert np.array_equal(asm.col_ptr, cp) and np.array_equal(asm.row_idx, ri)
    assert np.array_equal(bits(asm.residual), bits(res))
    nan = np.isnan(va)
    assert nan.any() and np.array_equal(np.isnan(asm.values), nan)
    assert np.array_equal(bits(asm.values[~nan]), bits(va[~nan]))
