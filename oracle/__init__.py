"""Parity oracle -- TEST INFRASTRUCTURE ONLY.

ctypes bindings to
  * ``oracle/build/liboracle.so``    -- the plain-C restatement of the reference hot path
                                        (``fibra_oracle.c``; always buildable), and
  * ``oracle/_ref/libfibra_ref.so``  -- the reference's own TUs compiled in place from
                                        /root/reference/proj/src (+ ``ref_shim.cpp``),
                                        present only where it was built.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product
(``paper_2306_09427_b200``) never does: it fails loudly when its CUDA library is missing.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfibra_ref.so")
REF_SRC = "/root/reference/proj"

STATUS = {0: "ok", 1: "config", 2: "kinematics", 3: "collapse", 4: "bad_dt", 5: "diverged",
          6: "not_converged", 7: "probe_failed", 8: "singular", 9: "unconverged_state",
          10: "nonfinite_stress", 11: "nonfinite_residual"}

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)
_bp = C.POINTER(C.c_uint8)


def build(ref: bool | None = None) -> None:
    """Compile the oracle (and oracle/_ref when the reference sources are present)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref is None:
        ref = os.path.isdir(REF_SRC)
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


class CNetwork(C.Structure):
    _fields_ = [("n_nodes", C.c_int), ("n_fibers", C.c_int), ("n_free", C.c_int),
                ("n_boundary", C.c_int), ("box_half", C.c_double), ("tol_bnd", C.c_double),
                ("max_ea", C.c_double), ("coords", _dp), ("fib_a", _ip), ("fib_b", _ip),
                ("area", _dp), ("modulus", _dp), ("rest_length", _dp),
                ("boundary_mask", _bp), ("boundary_nodes", _ip), ("packed_of_dof", _ip),
                ("dof_of_packed", _ip), ("packed_ref", _dp), ("fiber_dofs", _ip),
                ("node_lump", _dp)]


class CLaw(C.Structure):
    _fields_ = [("kind", C.c_int), ("ea_scale", C.c_double), ("nonlinearity", C.c_double),
                ("buckling_off", C.c_int)]


class CRelaxCfg(C.Structure):
    _fields_ = [("damping", C.c_double), ("tolerance", C.c_double),
                ("max_iterations", C.c_int64), ("dt_safety", C.c_double),
                ("density_scale", C.c_double)]


class CReport(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("residual", C.c_double), ("eps_eff", C.c_double),
                ("kinetic_fraction", C.c_double), ("dt", C.c_double), ("converged", C.c_int32),
                ("energy_drift", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class CState(C.Structure):
    _fields_ = [("u", _dp), ("v", _dp), ("a", _dp), ("f_int", _dp), ("f_damp", _dp),
                ("mass", _dp), ("inv_mass", _dp), ("t", _dp), ("iters", _lp),
                ("converged", _bp), ("n_free", C.c_int), ("n_dof", C.c_int)]


class CResponse(C.Structure):
    _fields_ = [("sigma", C.c_double * 6), ("spatial_c", C.c_double * 36),
                ("pk2", C.c_double * 6), ("material_a", C.c_double * 36),
                ("stress_asymmetry", C.c_double), ("base_report", CReport),
                ("solves", C.c_int32), ("relax_iterations", C.c_int64),
                ("failed_probe", C.c_int32)]


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        L = C.CDLL(ORACLE_SO)
        L.or_network_build.restype = C.c_int
        L.or_network_build.argtypes = [_dp, C.c_int, _ip, _ip, _dp, _dp, C.c_int, C.c_double,
                                       C.c_double, C.POINTER(CNetwork)]
        L.or_network_free.argtypes = [C.POINTER(CNetwork)]
        L.or_relax_solve.argtypes = [C.POINTER(CNetwork), C.POINTER(CLaw), _dp,
                                     C.POINTER(CRelaxCfg), CState, C.c_int, C.POINTER(CReport)]
        L.or_internal_forces_cfl.argtypes = [C.POINTER(CNetwork), C.POINTER(CLaw), _dp, _dp,
                                             _dp, _dp]
        L.or_homogenized_stress.argtypes = [C.POINTER(CNetwork), C.POINTER(CState), _dp, _dp, _dp]
        L.or_constitutive_response.argtypes = [C.POINTER(CNetwork), C.POINTER(CLaw), _dp,
                                               C.POINTER(CRelaxCfg), C.c_double, C.c_int,
                                               C.c_int, CState, C.POINTER(CResponse)]
        L.or_batch_response.argtypes = [C.POINTER(C.POINTER(CNetwork)), _ip, C.c_int, _lp,
                                        _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _lp, _bp, _ip,
                                        C.POINTER(CLaw), _dp, C.POINTER(CRelaxCfg), C.c_double,
                                        C.c_int, C.c_int, C.c_int, C.POINTER(CResponse), _ip]
        L.or_polar_decompose.argtypes = [_dp, _dp, _dp]
        L.or_eigen_sym3.argtypes = [_dp, _dp, _dp]
        L.or_libm.argtypes = [C.c_int, _dp, C.c_int64, _dp]
        L.or_pull_back_stress.argtypes = [_dp, _dp, _dp]
        L.or_push_forward_stiffness.argtypes = [_dp, _dp, _dp]
        L.or_material_stiffness_from_probes.argtypes = [_dp, _dp, _dp, C.c_double, _dp]
        L.or_norm2_sq.restype = C.c_double
        L.or_norm2_sq.argtypes = [C.c_int64, _dp]
        L.or_det.restype = C.c_double
        L.or_det.argtypes = [_dp]
        L.or_orientation_p2.restype = C.c_double
        L.or_orientation_p2.argtypes = [C.POINTER(CNetwork), _dp, _dp]
        _lib = L
    return _lib


# ----------------------------------------------------------------------------------
# configuration records (defaults = the reference's: relax.hpp:16-21, stiffness.hpp:13-14,
# network.hpp:28-32)
# ----------------------------------------------------------------------------------
@dataclass
class Law:
    kind: int = 0  # 0 linear, 1 exponential
    ea_scale: float = 1.0
    nonlinearity: float = 1.2
    buckling_off: bool = False

    def c(self):
        return CLaw(self.kind, self.ea_scale, self.nonlinearity, int(self.buckling_off))


@dataclass
class RelaxConfig:
    damping: float = 2.0
    tolerance: float = 1e-6
    max_iterations: int = 500000
    dt_safety: float = 0.8
    density_scale: float = 1.0

    def c(self):
        return CRelaxCfg(self.damping, self.tolerance, self.max_iterations, self.dt_safety,
                         self.density_scale)


class OracleError(RuntimeError):
    def __init__(self, code, what=""):
        super().__init__(f"{STATUS.get(code, code)} {what}".strip())
        self.code = code


class Network:
    """or_network (restated FiberNetwork, network.cpp:67-157)."""

    def __init__(self, coords, fib_a, fib_b, area=None, modulus=None, box_half=0.5,
                 tol_bnd=1e-6):
        coords = np.ascontiguousarray(coords, dtype=np.float64).reshape(-1, 3)
        fa = np.ascontiguousarray(fib_a, dtype=np.int32)
        fb = np.ascontiguousarray(fib_b, dtype=np.int32)
        m = len(fa)
        area = np.ones(m) if area is None else np.ascontiguousarray(area, dtype=np.float64)
        modulus = np.ones(m) if modulus is None else np.ascontiguousarray(modulus, np.float64)
        self.c = CNetwork()
        rc = lib().or_network_build(_ptr(coords, _dp), len(coords), _ptr(fa, _ip), _ptr(fb, _ip),
                                    _ptr(area, _dp), _ptr(modulus, _dp), m, box_half, tol_bnd,
                                    C.byref(self.c))
        if rc:
            raise OracleError(rc, "network construction")
        n, mm = self.c.n_nodes, self.c.n_fibers
        self.n_nodes, self.n_fibers, self.n_free = n, mm, self.c.n_free
        self.n_dof = 3 * n
        self.box_half = box_half
        self.coords = np.ctypeslib.as_array(self.c.coords, (3 * n,)).copy().reshape(-1, 3)
        self.fib_a = np.ctypeslib.as_array(self.c.fib_a, (mm,)).copy() if mm else np.zeros(0, np.int32)
        self.fib_b = np.ctypeslib.as_array(self.c.fib_b, (mm,)).copy() if mm else np.zeros(0, np.int32)
        self.area = area.copy()
        self.modulus = modulus.copy()
        self.rest_length = np.ctypeslib.as_array(self.c.rest_length, (mm,)).copy() if mm else np.zeros(0)
        self.boundary_nodes = np.ctypeslib.as_array(self.c.boundary_nodes, (self.c.n_boundary,)).copy()
        self.packed_of_dof = np.ctypeslib.as_array(self.c.packed_of_dof, (3 * n,)).copy()
        self.packed_ref = np.ctypeslib.as_array(self.c.packed_ref, (3 * n,)).copy()
        self.fiber_dofs = np.ctypeslib.as_array(self.c.fiber_dofs, (6 * mm,)).copy() if mm else np.zeros(0, np.int32)
        self.node_lump = np.ctypeslib.as_array(self.c.node_lump, (n,)).copy()
        self.max_ea = self.c.max_ea

    def __del__(self):
        try:
            lib().or_network_free(C.byref(self.c))
        except Exception:
            pass


class State:
    """Owning RveState (network.hpp:119-135) as numpy arrays."""

    def __init__(self, n_dof, n_free):
        self.n_dof, self.n_free = n_dof, n_free
        for k in ("u", "v", "a", "f_int", "f_damp", "mass", "inv_mass"):
            setattr(self, k, np.zeros(n_dof))
        self.t = np.zeros(1)
        self.iters = np.zeros(1, np.int64)
        self.converged = np.zeros(1, np.uint8)

    def c(self):
        return CState(*(_ptr(getattr(self, k), _dp) for k in
                        ("u", "v", "a", "f_int", "f_damp", "mass", "inv_mass", "t")),
                      _ptr(self.iters, _lp), _ptr(self.converged, _bp), self.n_free, self.n_dof)

    def copy(self):
        s = State(self.n_dof, self.n_free)
        for k in ("u", "v", "a", "f_int", "f_damp", "mass", "inv_mass", "t", "iters", "converged"):
            setattr(s, k, getattr(self, k).copy())
        return s


def _F(F):
    return np.ascontiguousarray(F, dtype=np.float64).reshape(9)


def relax_solve(net: Network, F, cfg: RelaxConfig = None, law: Law = None, state: State = None,
                warm_reuse: bool = False):
    """relax_solve (relax.cpp:93-199).  Fresh state + zero_interior when state is None."""
    cfg = cfg or RelaxConfig()
    law = law or Law()
    if state is None:
        state = State(net.n_dof, net.n_free)
    rep = CReport()
    F = _F(F)
    rc = lib().or_relax_solve(C.byref(net.c), C.byref(law.c()), _ptr(F, _dp), C.byref(cfg.c()),
                              state.c(), int(warm_reuse), C.byref(rep))
    if rc:
        raise OracleError(rc, "relax_solve")
    return state, rep.as_dict()


def homogenized_stress(net: Network, state: State, F):
    sig = np.zeros(6)
    asym = np.zeros(1)
    cs = state.c()
    F = _F(F)
    rc = lib().or_homogenized_stress(C.byref(net.c), C.byref(cs), _ptr(F, _dp), _ptr(sig, _dp),
                                     _ptr(asym, _dp))
    if rc:
        raise OracleError(rc, "homogenized_stress")
    return sig, float(asym[0])


def orientation_p2(net: Network, u, ref_dir) -> float:
    """orientation_p2 (network.cpp:398-415)."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    d = np.ascontiguousarray(ref_dir, dtype=np.float64)
    return float(lib().or_orientation_p2(C.byref(net.c), _ptr(u, _dp), _ptr(d, _dp)))


def internal_forces(net: Network, u, law: Law = None):
    law = law or Law()
    u = np.ascontiguousarray(u, dtype=np.float64)
    f = np.zeros(net.n_dof)
    rc = lib().or_internal_forces_cfl(C.byref(net.c), C.byref(law.c()), _ptr(u, _dp), _ptr(f, _dp),
                                      None, None)
    if rc:
        raise OracleError(rc, "internal_forces")
    return f


def polar_decompose(F):
    R = np.zeros(9)
    U = np.zeros(6)
    F = _F(F)
    rc = lib().or_polar_decompose(_ptr(F, _dp), _ptr(R, _dp), _ptr(U, _dp))
    if rc:
        raise OracleError(rc, "polar")
    return R.reshape(3, 3), U


def eigen_sym3(A):
    """Eigen 3.4.0 SelfAdjointEigenSolver<Matrix3d> restatement: (eigenvalues ascending,
    eigenvector columns)."""
    A = np.ascontiguousarray(np.asarray(A, dtype=np.float64).reshape(9))
    lam = np.zeros(3)
    Q = np.zeros(9)
    rc = lib().or_eigen_sym3(_ptr(A, _dp), _ptr(lam, _dp), _ptr(Q, _dp))
    if rc:
        raise OracleError(7, "eigen_sym3 NoConvergence")
    return lam, Q.reshape(3, 3)


def libm(which, x):
    """The host libm's exp (which 0) / expm1 (which 1), elementwise."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    lib().or_libm(int(which), _ptr(x, _dp), x.size, _ptr(out, _dp))
    return out


def norm2_sq(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    return lib().or_norm2_sq(len(x), _ptr(x, _dp))


def response_dict(r: CResponse):
    return {"sigma": np.array(r.sigma[:]), "spatial_c": np.array(r.spatial_c[:]).reshape(6, 6),
            "pk2": np.array(r.pk2[:]), "material_a": np.array(r.material_a[:]).reshape(6, 6),
            "stress_asymmetry": r.stress_asymmetry, "base_report": r.base_report.as_dict(),
            "solves": r.solves, "relax_iterations": r.relax_iterations,
            "failed_probe": r.failed_probe}


def constitutive_response(net: Network, F, relax_cfg=None, law=None, fd_rel_step=1e-5,
                          reuse_warm=True, want_tangent=True, state: State = None):
    relax_cfg = relax_cfg or RelaxConfig()
    law = law or Law()
    if state is None:
        state = State(net.n_dof, net.n_free)
    out = CResponse()
    F = _F(F)
    rc = lib().or_constitutive_response(C.byref(net.c), C.byref(law.c()), _ptr(F, _dp),
                                        C.byref(relax_cfg.c()), fd_rel_step, int(reuse_warm),
                                        int(want_tangent), state.c(), C.byref(out))
    if rc:
        raise OracleError(rc, "constitutive_response")
    return response_dict(out), state


@dataclass
class PackedStates:
    """PackedStates (batch.hpp:20-31): CRS offsets + shared value arrays."""
    offsets: np.ndarray
    n_free: np.ndarray
    arrays: dict = field(default_factory=dict)

    @staticmethod
    def fresh(nets, entry_of_point):
        n = len(entry_of_point)
        nd = np.array([nets[e].n_dof for e in entry_of_point], np.int64)
        offs = np.zeros(n + 1, np.int64)
        offs[1:] = np.cumsum(nd)
        ps = PackedStates(offs, np.array([nets[e].n_free for e in entry_of_point], np.int32))
        tot = int(offs[-1])
        for k in ("u", "v", "a", "f_int", "f_damp", "mass", "inv_mass"):
            ps.arrays[k] = np.zeros(tot)
        ps.arrays["t"] = np.zeros(n)
        ps.arrays["iters"] = np.zeros(n, np.int64)
        ps.arrays["converged"] = np.zeros(n, np.uint8)
        return ps


def batch_response(nets, entry_of_point, states: PackedStates, F, relax_cfg=None, law=None,
                   fd_rel_step=1e-5, reuse_warm=True, want_tangent=True, n_threads=1):
    """batch_response (batch.cpp:155-187).  Returns (responses list, status array)."""
    relax_cfg = relax_cfg or RelaxConfig()
    law = law or Law()
    eop = np.ascontiguousarray(entry_of_point, dtype=np.int32)
    n = len(eop)
    F = np.ascontiguousarray(F, dtype=np.float64).reshape(n, 9)
    arr = (C.POINTER(CNetwork) * len(nets))(*[C.pointer(nt.c) for nt in nets])
    out = (CResponse * max(n, 1))()
    status = np.zeros(n, np.int32)
    A = states.arrays
    rc = lib().or_batch_response(arr, _ptr(eop, _ip), n, _ptr(states.offsets, _lp),
                                 *(_ptr(A[k], _dp) for k in ("u", "v", "a", "f_int", "f_damp",
                                                             "mass", "inv_mass", "t")),
                                 _ptr(A["iters"], _lp), _ptr(A["converged"], _bp),
                                 _ptr(states.n_free, _ip), C.byref(law.c()), _ptr(F, _dp),
                                 C.byref(relax_cfg.c()), fd_rel_step, int(reuse_warm),
                                 int(want_tangent), n_threads, out, _ptr(status, _ip))
    if rc:
        raise OracleError(rc, "batch_response")
    return [response_dict(out[p]) for p in range(n)], status


# ----------------------------------------------------------------------------------
# oracle/_ref: the reference's own compiled TUs
# ----------------------------------------------------------------------------------
_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        L = C.CDLL(REF_SO)
        L.ref_generate.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                                   C.c_double, _dp, C.c_double, C.c_double, C.c_double,
                                   C.c_double, C.c_uint64, C.POINTER(C.c_void_p)]
        L.ref_network_from_arrays.argtypes = [_dp, C.c_int, _ip, _ip, _dp, _dp, C.c_int,
                                              C.c_double, C.c_double, C.POINTER(C.c_void_p)]
        L.ref_network_read.argtypes = [C.c_char_p, C.c_double, C.c_double, C.POINTER(C.c_void_p)]
        L.ref_network_write.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_network_free.argtypes = [C.c_void_p]
        L.ref_network_sizes.argtypes = [C.c_void_p] + [C.POINTER(C.c_int)] * 4
        L.ref_network_export.argtypes = [C.c_void_p, _dp, _ip, _ip, _dp, _dp, _dp, _ip, _ip, _dp,
                                         _ip, _dp, _dp]
        L.ref_relax_solve.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_int, _dp,
                                      C.POINTER(CRelaxCfg), _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                      _dp, _lp, _bp, C.c_int, C.POINTER(CReport)]
        L.ref_homogenized_stress.argtypes = [C.c_void_p, _dp, _dp, C.c_int, _dp, _dp, _dp]
        L.ref_orientation_p2.restype = C.c_double
        L.ref_orientation_p2.argtypes = [C.c_void_p, _dp, _dp]
        L.ref_internal_forces.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_int,
                                          _dp, _dp]
        L.ref_batch_stress.argtypes = [C.c_void_p, C.c_int, _dp, C.c_int, C.c_double, C.c_double,
                                       C.c_int, C.POINTER(CRelaxCfg), C.c_int, _dp, _lp, _ip]
        L.ref_batch_response.argtypes = [C.POINTER(C.c_void_p), _ip, C.c_int, _dp, C.c_int,
                                         C.c_double, C.c_double, C.c_int,
                                         C.POINTER(CRelaxCfg), C.c_double, C.c_int, C.c_int,
                                         C.c_int, _dp, _dp, _lp, _lp, _ip, _ip, _ip]
        L.ref_last_error.restype = C.c_char_p
        _ref = L
    return _ref


class RefNetwork:
    """Handle to a reference fibra::FiberNetwork living in oracle/_ref."""

    def __init__(self, handle):
        self.h = C.c_void_p(handle)
        n, m, nf, nb = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        ref().ref_network_sizes(self.h, C.byref(n), C.byref(m), C.byref(nf), C.byref(nb))
        self.n_nodes, self.n_fibers, self.n_free, self.n_boundary = n.value, m.value, nf.value, nb.value
        self.n_dof = 3 * self.n_nodes
        N, M = self.n_nodes, self.n_fibers
        self.coords = np.zeros(3 * N)
        self.fib_a = np.zeros(M, np.int32)
        self.fib_b = np.zeros(M, np.int32)
        self.area = np.zeros(M)
        self.modulus = np.zeros(M)
        self.rest_length = np.zeros(M)
        self.boundary_nodes = np.zeros(self.n_boundary, np.int32)
        self.packed_of_dof = np.zeros(3 * N, np.int32)
        self.packed_ref = np.zeros(3 * N)
        self.fiber_dofs = np.zeros(6 * M, np.int32)
        self.node_lump = np.zeros(N)
        me = np.zeros(1)
        ref().ref_network_export(self.h, _ptr(self.coords, _dp), _ptr(self.fib_a, _ip),
                                 _ptr(self.fib_b, _ip), _ptr(self.area, _dp),
                                 _ptr(self.modulus, _dp), _ptr(self.rest_length, _dp),
                                 _ptr(self.boundary_nodes, _ip), _ptr(self.packed_of_dof, _ip),
                                 _ptr(self.packed_ref, _dp), _ptr(self.fiber_dofs, _ip),
                                 _ptr(self.node_lump, _dp), _ptr(me, _dp))
        self.coords = self.coords.reshape(-1, 3)
        self.max_ea = float(me[0])

    def __del__(self):
        try:
            ref().ref_network_free(self.h)
        except Exception:
            pass

    def write(self, path):
        rc = ref().ref_network_write(self.h, str(path).encode())
        if rc:
            raise OracleError(rc, ref().ref_last_error().decode())


def ref_generate(style="knn", nodes=60, fibers=200, half_length=0.3, merge_radius=0.05,
                 neighbors=8, align_bias=0.0, align_axis=(1.0, 0.0, 0.0), area=1.0,
                 modulus=1.0, box_half=0.5, tol_bnd=1e-6, seed=1) -> RefNetwork:
    """Reference generate_network (netgen.cpp:276-285), NetGenSpec defaults netgen.hpp:18-33."""
    h = C.c_void_p()
    ax = np.array(align_axis, dtype=np.float64)
    rc = ref().ref_generate(0 if style == "segments" else 1, nodes, fibers, half_length,
                            merge_radius, neighbors, align_bias, _ptr(ax, _dp), area, modulus,
                            box_half, tol_bnd, seed, C.byref(h))
    if rc:
        raise OracleError(rc, ref().ref_last_error().decode())
    return RefNetwork(h.value)


def ref_read(path, box_half=0.5, tol_bnd=1e-6) -> RefNetwork:
    h = C.c_void_p()
    rc = ref().ref_network_read(str(path).encode(), box_half, tol_bnd, C.byref(h))
    if rc:
        raise OracleError(rc, ref().ref_last_error().decode())
    return RefNetwork(h.value)


def ref_relax_solve(rnet: RefNetwork, F, cfg: RelaxConfig = None, law: Law = None,
                    state: State = None, warm_reuse=False):
    cfg = cfg or RelaxConfig()
    law = law or Law()
    if state is None:
        state = State(rnet.n_dof, rnet.n_free)
    rep = CReport()
    F = _F(F)
    rc = ref().ref_relax_solve(rnet.h, law.kind, law.ea_scale, law.nonlinearity,
                               int(law.buckling_off), _ptr(F, _dp), C.byref(cfg.c()),
                               *(_ptr(getattr(state, k), _dp) for k in
                                 ("u", "v", "a", "f_int", "f_damp", "mass", "inv_mass", "t")),
                               _ptr(state.iters, _lp), _ptr(state.converged, _bp),
                               int(warm_reuse), C.byref(rep))
    if rc:
        raise OracleError(rc, ref().ref_last_error().decode())
    return state, rep.as_dict()


def ref_homogenized_stress(rnet: RefNetwork, state: State, F):
    sig = np.zeros(6)
    asym = np.zeros(1)
    F = _F(F)
    rc = ref().ref_homogenized_stress(rnet.h, _ptr(state.u, _dp), _ptr(state.f_int, _dp),
                                      int(state.converged[0]), _ptr(F, _dp), _ptr(sig, _dp),
                                      _ptr(asym, _dp))
    if rc:
        raise OracleError(rc, ref().ref_last_error().decode())
    return sig, float(asym[0])


def ref_orientation_p2(rnet: RefNetwork, u, ref_dir) -> float:
    u = np.ascontiguousarray(u, dtype=np.float64)
    d = np.ascontiguousarray(ref_dir, dtype=np.float64)
    return float(ref().ref_orientation_p2(rnet.h, _ptr(u, _dp), _ptr(d, _dp)))


def ref_batch_stress(rnet: RefNetwork, F, cfg: RelaxConfig = None, law: Law = None, workers=1):
    cfg = cfg or RelaxConfig()
    law = law or Law()
    F = np.ascontiguousarray(F, dtype=np.float64).reshape(-1, 9)
    n = len(F)
    sig = np.zeros((n, 6))
    iters = np.zeros(n, np.int64)
    status = np.zeros(n, np.int32)
    rc = ref().ref_batch_stress(rnet.h, n, _ptr(F, _dp), law.kind, law.ea_scale,
                                law.nonlinearity, int(law.buckling_off), C.byref(cfg.c()),
                                workers, _ptr(sig, _dp), _ptr(iters, _lp), _ptr(status, _ip))
    if rc:
        raise OracleError(rc, ref().ref_last_error().decode())
    return sig, iters, status


def ref_batch_response(rnets, entry_of_point, F, cfg: RelaxConfig = None, law: Law = None,
                       fd_rel_step=1e-5, reuse_warm=True, want_tangent=True, workers=1):
    """constitutive_response per point (stiffness.cpp:153-175) with every DR solve and
    homogenized stress from the reference's compiled code (ref_shim.cpp), fresh states.
    Returns a dict of arrays: sigma (n,6), spatial_c (n,36), base_iterations,
    relax_iterations, solves, failed_probe, status."""
    cfg = cfg or RelaxConfig()
    law = law or Law()
    F = np.ascontiguousarray(F, dtype=np.float64).reshape(-1, 9)
    n = len(F)
    eop = np.ascontiguousarray(entry_of_point, dtype=np.int32)
    handles = (C.c_void_p * len(rnets))(*[r.h.value for r in rnets])
    out = {"sigma": np.zeros((n, 6)), "spatial_c": np.zeros((n, 36)),
           "base_iterations": np.zeros(n, np.int64), "relax_iterations": np.zeros(n, np.int64),
           "solves": np.zeros(n, np.int32), "failed_probe": np.zeros(n, np.int32),
           "status": np.zeros(n, np.int32)}
    rc = ref().ref_batch_response(handles, _ptr(eop, _ip), n, _ptr(F, _dp), law.kind,
                                  law.ea_scale, law.nonlinearity, int(law.buckling_off),
                                  C.byref(cfg.c()), fd_rel_step, int(reuse_warm),
                                  int(want_tangent), workers,
                                  *(_ptr(out[k], t) for k, t in
                                    (("sigma", _dp), ("spatial_c", _dp),
                                     ("base_iterations", _lp), ("relax_iterations", _lp),
                                     ("solves", _ip), ("failed_probe", _ip), ("status", _ip))))
    if rc:
        raise OracleError(rc, ref().ref_last_error().decode())
    return out


def network_from_ref(rnet: RefNetwork, box_half=0.5, tol_bnd=1e-6) -> Network:
    return Network(rnet.coords, rnet.fib_a, rnet.fib_b, rnet.area, rnet.modulus, box_half, tol_bnd)


# ----------------------------------------------------------------------------------
# macro assembly (macrofem.cpp:41-187): the checker of the device assembly
# ----------------------------------------------------------------------------------
def tet_geom(coords, tet):
    """b_matrix (macrofem.cpp:41-60) -> (grad[4,3], volume)."""
    c = np.ascontiguousarray(coords, dtype=np.float64)
    n = np.ascontiguousarray(tet, dtype=np.int32)
    g = np.zeros(12)
    v = C.c_double(0)
    L = lib()
    L.or_tet_geom.argtypes = [_dp, _ip, _dp, C.POINTER(C.c_double)]
    rc = L.or_tet_geom(_ptr(c, _dp), _ptr(n, _ip), _ptr(g, _dp), C.byref(v))
    if rc:
        raise OracleError(rc, "b_matrix")
    return g.reshape(4, 3), v.value


def assemble(tets, coords, sigma, c66, free_of_dof, n_free, f_ext=None):
    """assemble (macrofem.cpp:104-187) -> (residual, col_ptr, row_idx, values): the
    free x free stiffness in Eigen's compressed column-major layout.  Element errors raise
    OracleError with .element set to the first failing element."""
    tets = np.ascontiguousarray(tets, dtype=np.int32).reshape(-1, 4)
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    sigma = np.ascontiguousarray(sigma, dtype=np.float64).reshape(-1, 6)
    c66 = np.ascontiguousarray(c66, dtype=np.float64).reshape(-1, 36)
    fod = np.ascontiguousarray(free_of_dof, dtype=np.int32)
    ne = len(tets)
    cap = max(1, 144 * ne)
    res = np.zeros(n_free)
    cp = np.zeros(n_free + 1, np.int64)
    ri = np.zeros(cap, np.int32)
    va = np.zeros(cap)
    nnz = C.c_int64(0)
    bad = C.c_int32(-1)
    fe = None if f_ext is None else np.ascontiguousarray(f_ext, dtype=np.float64)
    L = lib()
    L.or_assemble.argtypes = [_ip, C.c_int32, _dp, _dp, _dp, _ip, C.c_int32, _dp, _dp, _lp,
                              _ip, _dp, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
    rc = L.or_assemble(_ptr(tets, _ip), ne, _ptr(coords, _dp), _ptr(sigma, _dp),
                       _ptr(c66, _dp), _ptr(fod, _ip), n_free,
                       None if fe is None else _ptr(fe, _dp), _ptr(res, _dp), _ptr(cp, _lp),
                       _ptr(ri, _ip), _ptr(va, _dp), cap, C.byref(nnz), C.byref(bad))
    if rc:
        err = OracleError(rc, f"assemble (element {bad.value})")
        err.element = bad.value
        raise err
    k = nnz.value
    return res, cp, ri[:k].copy(), va[:k].copy()
