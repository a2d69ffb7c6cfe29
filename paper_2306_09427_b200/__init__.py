"""B200-native batched fiber-network RVE solver (MuMFiM hot path, arXiv 2306.09427).

Python mirror of the reference's batched-RVE interface (reference
proj/include/fibra/batch.hpp:20-129, network.hpp, relax.hpp, stiffness.hpp, netgen.hpp):
same names, argument meaning and error behaviour, so a caller of
``fibra::batch_response`` finds the same call here::

    lib = RveLibrary([generate_network(NetGenSpec(style="knn", nodes=375, fibers=1000,
                                                  neighbors=10), seed=1)])
    states, assign = init_batch(np.zeros(n, np.int32), lib, seed=7)
    br = batch_response(lib, assign, states, FiberLaw(), F, RelaxConfig(), StiffnessConfig())

Every solve runs in the sm_100a CUDA library ``lib/libfibra_b200.so`` through the C-ABI of
``include/fibra_cuda.h``.  There is no CPU fallback: without the library or a B200 the
calls raise.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _capi
from ._capi import ptr as _ptr

__all__ = [
    "Error", "ConfigError", "KinematicsError", "SolverError", "IoError", "FiberLaw",
    "RelaxConfig", "StiffnessConfig", "NetGenSpec", "FiberNetwork", "generate_network",
    "RveLibrary", "BatchAssignment", "PackedStates", "init_batch", "PointResponse",
    "ResponseStats", "BatchResult", "DeviceBatch", "batch_response", "NetworkBatchProvider",
    "ProviderResult",
]


# ---- errors (error.hpp:8-28) ---------------------------------------------------------
class Error(RuntimeError):
    pass


class KinematicsError(Error):
    pass


class SolverError(Error):
    pass


class IoError(Error):
    pass


class ConfigError(Error):
    pass


class CudaError(Error):
    pass


def _raise(code: int, what: str):
    cls = {1: ConfigError, 2: KinematicsError, 22: IoError, 20: CudaError, 21: ConfigError}.get(
        code, SolverError)
    raise cls(what or _capi.STATUS_NAMES.get(code, str(code)))


# ---- configuration records -------------------------------------------------------------
@dataclass
class FiberLaw:  # network.hpp:27-38
    kind: str = "linear"  # "linear" | "exponential"
    ea_scale: float = 1.0
    nonlinearity: float = 1.2
    buckling_off: bool = False

    def c(self) -> _capi.Law:
        if self.kind not in ("linear", "exponential"):
            raise ConfigError(f"unknown fiber law '{self.kind}'")
        return _capi.Law(0 if self.kind == "linear" else 1, self.ea_scale, self.nonlinearity,
                         int(self.buckling_off))


@dataclass
class RelaxConfig:  # relax.hpp:15-26
    damping: float = 2.0
    tolerance: float = 1e-6
    max_iterations: int = 500000
    dt_safety: float = 0.8
    density_scale: float = 1.0
    energy_check: bool = False

    def c(self) -> _capi.RelaxCfg:
        return _capi.RelaxCfg(self.damping, self.tolerance, self.max_iterations,
                              self.dt_safety, self.density_scale, int(self.energy_check))


@dataclass
class StiffnessConfig:  # stiffness.hpp:12-17
    fd_rel_step: float = 1e-5
    reuse_warm: bool = True

    def c(self) -> _capi.StiffCfg:
        return _capi.StiffCfg(self.fd_rel_step, int(self.reuse_warm))


@dataclass
class NetGenSpec:  # netgen.hpp:16-33
    style: str = "segments"
    fibers: int = 200
    nodes: int = 60
    half_length: float = 0.3
    merge_radius: float = 0.05
    neighbors: int = 8
    align_bias: float = 0.0
    align_axis: Sequence[float] = (1.0, 0.0, 0.0)
    fiber_area: float = 1.0
    fiber_modulus: float = 1.0
    box_half: float = 0.5
    tol_bnd: float = 1e-6

    def c(self) -> _capi.NetgenSpec:
        if self.style not in ("segments", "knn"):
            raise ConfigError(f"unknown netgen style '{self.style}'")
        return _capi.NetgenSpec(0 if self.style == "segments" else 1, self.fibers, self.nodes,
                                self.half_length, self.merge_radius, self.neighbors,
                                self.align_bias, (C.c_double * 3)(*self.align_axis),
                                self.fiber_area, self.fiber_modulus, self.box_half,
                                self.tol_bnd)


# ---- networks ---------------------------------------------------------------------------
class FiberNetwork:
    """Immutable RVE network (network.hpp:55-101), built by the library's host C++."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        d = _capi.NetDesc()
        _capi.load().fibra_network_describe(self._h, C.byref(d))
        self._desc = d
        N, M = d.n_nodes, d.n_fibers
        cp = lambda p, n, shape=None: (np.ctypeslib.as_array(p, (n,)).copy() if n else
                                       np.zeros(0, np.float64 if isinstance(p, _capi._dp) else np.int32))
        self.n_nodes, self.n_fibers, self.n_free = N, M, d.n_free
        self.n_dof = 3 * N
        self.box_half = d.box_half
        self.max_ea = d.max_ea
        self.coords = np.ctypeslib.as_array(d.coords, (3 * N,)).copy().reshape(N, 3)
        self.fiber_nodes = (np.ctypeslib.as_array(d.fiber_nodes, (2 * M,)).copy().reshape(M, 2)
                            if M else np.zeros((0, 2), np.int32))
        self.fiber_area = cp(d.fiber_area, M)
        self.fiber_modulus = cp(d.fiber_modulus, M)
        self.packed_of_dof = np.ctypeslib.as_array(d.packed_of_dof, (3 * N,)).copy()
        self.packed_ref_coords = np.ctypeslib.as_array(d.packed_ref, (3 * N,)).copy()
        self.fiber_packed_dofs = cp(d.fiber_packed_dofs, 6 * M)
        self.rest_lengths = cp(d.rest_length, M)
        self.node_lumping = np.ctypeslib.as_array(d.node_lump, (N,)).copy()
        self.boundary_nodes = np.ctypeslib.as_array(d.boundary_nodes, (d.n_boundary,)).copy()

    @staticmethod
    def _check(rc: int):
        if rc:
            _raise(rc, _capi.load().fibra_host_last_error().decode())

    @classmethod
    def from_arrays(cls, coords, fiber_nodes, area=None, modulus=None, box_half=0.5,
                    tol_bnd=1e-6) -> "FiberNetwork":
        coords = np.ascontiguousarray(coords, dtype=np.float64).reshape(-1, 3)
        fn = np.ascontiguousarray(fiber_nodes, dtype=np.int32).reshape(-1, 2)
        m = len(fn)
        area = np.ones(m) if area is None else np.ascontiguousarray(area, dtype=np.float64)
        modulus = np.ones(m) if modulus is None else np.ascontiguousarray(modulus, np.float64)
        h = C.c_void_p()
        cls._check(_capi.load().fibra_network_create(_ptr(coords, _capi._dp), len(coords),
                                                     _ptr(fn, _capi._ip), _ptr(area, _capi._dp),
                                                     _ptr(modulus, _capi._dp), m, box_half,
                                                     tol_bnd, C.byref(h)))
        return cls(h)

    @classmethod
    def read_file(cls, path, box_half=0.5, tol_bnd=1e-6) -> "FiberNetwork":
        h = C.c_void_p()
        cls._check(_capi.load().fibra_network_read(str(path).encode(), box_half, tol_bnd,
                                                   C.byref(h)))
        return cls(h)

    def write_file(self, path) -> None:
        self._check(_capi.load().fibra_network_write(self._h, str(path).encode()))

    def desc(self) -> _capi.NetDesc:
        return self._desc

    def __del__(self):
        try:
            if self._h:
                _capi.load(build_if_missing=False).fibra_network_free(self._h)
                self._h = None
        except Exception:
            pass


def generate_network(spec: NetGenSpec, seed: int) -> FiberNetwork:
    """generate_network (netgen.cpp:276-285) -- output-identical, grid-accelerated."""
    h = C.c_void_p()
    FiberNetwork._check(_capi.load().fibra_network_generate(C.byref(spec.c()), seed, C.byref(h)))
    return FiberNetwork(h)


def generate_lattice_network(n_side: int, fibers: int, seed: int, jitter: float = 0.25,
                             fiber_area: float = 1.0, fiber_modulus: float = 1.0,
                             box_half: float = 0.5, tol_bnd: float = 1e-6) -> FiberNetwork:
    """Builder-side jittered lattice for config-4 sized RVEs (~50k fibers; the reference's
    knn generator fails there).  n_side^3 nodes, face nodes exactly on the box,
    every axis bond plus seeded face diagonals up to `fibers`."""
    h = C.c_void_p()
    FiberNetwork._check(_capi.load().fibra_network_generate_lattice(
        int(n_side), int(fibers), float(jitter), float(fiber_area), float(fiber_modulus),
        float(box_half), float(tol_bnd), int(seed), C.byref(h)))
    return FiberNetwork(h)


# ---- library / assignment / packed states (batch.hpp:20-61) -----------------------------
@dataclass
class RveLibrary:
    entries: List[FiberNetwork] = field(default_factory=list)
    policy: str = "random"  # "random" | "per_region" | "explicit"
    region_map: Dict[int, int] = field(default_factory=dict)
    explicit_assignment: List[int] = field(default_factory=list)

    def validate(self):  # batch.cpp:31-45
        if not self.entries:
            raise ConfigError("RVE library is empty")
        n = len(self.entries)
        if self.policy == "per_region":
            if not self.region_map:
                raise ConfigError("per-region policy needs a region map")
            for tag, e in self.region_map.items():
                if e < 0 or e >= n:
                    raise ConfigError(f"region map entry for tag {tag} is out of range")
        if self.policy == "explicit":
            for e in self.explicit_assignment:
                if e < 0 or e >= n:
                    raise ConfigError("explicit assignment out of range")


@dataclass
class BatchAssignment:
    entry_of_point: np.ndarray


@dataclass
class PackedStates:
    offsets: np.ndarray
    u: np.ndarray
    v: np.ndarray
    a: np.ndarray
    f_int: np.ndarray
    f_damp: np.ndarray
    mass: np.ndarray
    inv_mass: np.ndarray
    t: np.ndarray
    iters: np.ndarray
    converged: np.ndarray
    n_free: np.ndarray

    def n_points(self) -> int:
        return len(self.t)

    def total_dofs(self) -> int:
        return int(self.offsets[-1]) if len(self.offsets) else 0

    def view(self, p: int) -> dict:  # PackedStates::view batch.cpp:13-29
        lo, hi = int(self.offsets[p]), int(self.offsets[p + 1])
        d = {k: getattr(self, k)[lo:hi] for k in ("u", "v", "a", "f_int", "f_damp", "mass",
                                                  "inv_mass")}
        d.update(t=self.t[p:p + 1], iters=self.iters[p:p + 1],
                 converged=self.converged[p:p + 1], n_free=int(self.n_free[p]))
        return d


def init_batch(region_of_point, library: RveLibrary, seed: int):
    """init_batch (batch.cpp:94-145): deterministic assignment + zero-filled states."""
    library.validate()
    regions = np.asarray(region_of_point, dtype=np.int32)
    n = len(regions)
    eop = np.zeros(n, np.int32)
    if library.policy == "random":
        if n:
            rc = _capi.load().fibra_assign_random(seed, n, len(library.entries),
                                                  _ptr(eop, _capi._ip))
            if rc:
                _raise(rc, "assignment")
    elif library.policy == "per_region":
        for p, r in enumerate(regions):
            if int(r) not in library.region_map:
                raise ConfigError(f"no library entry mapped for region {int(r)}")
            eop[p] = library.region_map[int(r)]
    elif library.policy == "explicit":
        if n > len(library.explicit_assignment):
            raise ConfigError("explicit assignment list shorter than point count")
        eop[:] = library.explicit_assignment[:n]
    else:
        raise ConfigError(f"unknown assignment policy '{library.policy}'")
    nd = np.array([library.entries[e].n_dof for e in eop], np.int64)
    offsets = np.zeros(n + 1, np.int64)
    offsets[1:] = np.cumsum(nd)
    tot = int(offsets[-1])
    z = lambda: np.zeros(tot)
    st = PackedStates(offsets, z(), z(), z(), z(), z(), z(), z(), np.zeros(n), np.zeros(n, np.int64),
                      np.zeros(n, np.uint8),
                      np.array([library.entries[e].n_free for e in eop], np.int32))
    return st, BatchAssignment(eop)


# ---- results ----------------------------------------------------------------------------
@dataclass
class PointResponse:  # macrofem.hpp:48-51
    sigma: np.ndarray      # (6,) xx yy zz yz xz xy
    spatial_c: np.ndarray  # (6,6) Mandel


@dataclass
class ResponseStats:  # stiffness.hpp:19-23
    solves: int = 0
    relax_iterations: int = 0
    failed_probe: int = -1


@dataclass
class BatchResult:  # batch.hpp:64-69
    responses: List[PointResponse]
    stats: List[ResponseStats]
    base_reports: List[dict]
    failed: List[int]
    records: np.ndarray = None  # raw fibra_point_result records (structured array)


RESULT_DTYPE = np.dtype(_capi.PointResult)


def _to_result(rec: np.ndarray) -> BatchResult:
    status = rec["status"]
    responses, stats, reports = [], [], []
    for p in range(len(rec)):
        r = rec[p]
        responses.append(PointResponse(np.array(r["sigma"]), np.array(r["spatial_c"]).reshape(6, 6)))
        stats.append(ResponseStats(int(r["solves"]), int(r["relax_iterations"]),
                                   int(r["failed_probe"]) if status[p] == 0 else -1))
        br = r["base_report"]
        reports.append({k: br[k].item() for k in br.dtype.names if not k.startswith("reserved")})
    failed = [int(p) for p in np.nonzero(status)[0]]
    return BatchResult(responses, stats, reports, failed, rec)


# ---- device context ---------------------------------------------------------------------
SCHED_BATCH, SCHED_STRAIN, SCHED_HINT = 0, 1, 2  # fibra_cuda_set_schedule modes


class DeviceBatch:
    """A CUDA context holding one RveLibrary in HBM and the PackedStates of one assignment.

    Device-resident across calls (the warm state stays in HBM); the reference semantics of a
    host-owned PackedStates are provided by ``batch_response`` which uploads/downloads it.
    """

    def __init__(self, library: RveLibrary, assignment: BatchAssignment, device: int = 0,
                 stream: Optional[int] = None, devices: Optional[Sequence[int]] = None):
        """``devices``: several GPUs of this process (fibra_cuda_open_devices): the library
        is replicated, the points are sharded by longest-processing-time on their cost, and
        the records come back through one NCCL all-gather; device pointers of
        ``solve_device`` then live on ``devices[0]``."""
        L = _capi.load()
        self._L = L
        self._ctx = C.c_void_p()
        self.devices = [int(d) for d in devices] if devices else [int(device)]
        if len(self.devices) > 1:
            devs = np.ascontiguousarray(self.devices, dtype=np.int32)
            self._check(L.fibra_cuda_open_devices(_ptr(devs, _capi._ip), len(devs),
                                                  C.byref(self._ctx)), ctx=False)
        else:
            self._check(L.fibra_cuda_open(self.devices[0], C.byref(self._ctx)), ctx=False)
        if stream:
            self._check(L.fibra_cuda_set_stream(self._ctx, C.c_void_p(stream)))
        self.library = library
        descs = (_capi.NetDesc * len(library.entries))(*[e.desc() for e in library.entries])
        self._check(L.fibra_cuda_upload_library(self._ctx, descs, len(library.entries)))
        self.entry_of_point = np.ascontiguousarray(assignment.entry_of_point, dtype=np.int32)
        self.n_points = len(self.entry_of_point)
        self._check(L.fibra_cuda_bind_points(self._ctx, _ptr(self.entry_of_point, _capi._ip),
                                             self.n_points))
        self._out = np.zeros(max(self.n_points, 1), RESULT_DTYPE)

    def _check(self, rc: int, ctx: bool = True):
        if rc:
            msg = self._L.fibra_cuda_last_error(self._ctx).decode() if ctx else "fibra_cuda_open"
            _raise(rc, msg)

    def reset_states(self):
        self._check(self._L.fibra_cuda_reset_states(self._ctx))

    def orientation(self, points, ref_dir) -> np.ndarray:
        """orientation_p2 (network.cpp:398-415) of the device-resident states of `points`."""
        pts = np.ascontiguousarray(points, dtype=np.int32).reshape(-1)
        d = np.ascontiguousarray(ref_dir, dtype=np.float64).reshape(3)
        out = np.zeros(max(len(pts), 1))
        self._check(self._L.fibra_cuda_orientation(self._ctx, _ptr(pts, _capi._ip), len(pts),
                                                   _ptr(d, _capi._dp), _ptr(out, _capi._dp)))
        return out[:len(pts)]

    def entry_kernel(self, entry: int) -> dict:
        """Kernel shape of a library entry: cluster size (1 = one CTA per RVE) and per-CTA
        threads / fibers per thread / nodes per thread."""
        out = np.zeros(4, np.int32)
        self._check(self._L.fibra_cuda_entry_kernel(self._ctx, int(entry), _ptr(out, _capi._ip)))
        return {"cluster": int(out[0]), "threads": int(out[1]), "fibers_per_thread": int(out[2]),
                "nodes_per_thread": int(out[3])}

    def set_schedule(self, mode: int, cost_hint=None):
        """Start order of base solves (SCHED_BATCH / SCHED_STRAIN / SCHED_HINT); results do
        not depend on it, only the makespan does.  ``cost_hint``: one cost per point, larger
        first (e.g. the previous call's relax_iterations)."""
        hint = None
        if mode == SCHED_HINT:
            hint = np.ascontiguousarray(cost_hint, dtype=np.float64)
            if hint.shape != (self.n_points,):
                raise ConfigError("cost_hint needs one value per point")
        self._check(self._L.fibra_cuda_set_schedule(
            self._ctx, int(mode), None if hint is None else _ptr(hint, _capi._dp)))

    def upload_states(self, st: PackedStates):
        self._check(self._L.fibra_cuda_upload_states(
            self._ctx, _ptr(st.u, _capi._dp), _ptr(st.t, _capi._dp), _ptr(st.iters, _capi._lp),
            _ptr(st.converged, _capi._bp)))

    def download_states(self, st: PackedStates):
        self._check(self._L.fibra_cuda_download_states(
            self._ctx, *(_ptr(getattr(st, k), _capi._dp) for k in
                         ("u", "v", "a", "f_int", "f_damp", "mass", "inv_mass", "t")),
            _ptr(st.iters, _capi._lp), _ptr(st.converged, _capi._bp)))

    def solve(self, deformation, law: FiberLaw = None, relax_cfg: RelaxConfig = None,
              stiff_cfg: StiffnessConfig = None, want_tangent: bool = True) -> np.ndarray:
        """All points, host arrays in and out; returns fibra_point_result records."""
        law = law or FiberLaw()
        relax_cfg = relax_cfg or RelaxConfig()
        stiff_cfg = stiff_cfg or StiffnessConfig()
        F = np.ascontiguousarray(deformation, dtype=np.float64).reshape(-1, 9)
        if len(F) != self.n_points:
            raise ConfigError("one deformation gradient per point is required")
        out = self._out
        self._check(self._L.fibra_cuda_solve(
            self._ctx, _ptr(F, _capi._dp), C.byref(law.c()), C.byref(relax_cfg.c()),
            C.byref(stiff_cfg.c()), int(want_tangent),
            out.ctypes.data_as(C.POINTER(_capi.PointResult))))
        return out[:self.n_points].copy()

    def solve_device(self, F_dev_ptr: int, out_dev_ptr: int, law: FiberLaw = None,
                     relax_cfg: RelaxConfig = None, stiff_cfg: StiffnessConfig = None,
                     want_tangent: bool = True):
        """Asynchronous solve on device-resident F / result buffers (raw device pointers)."""
        law = law or FiberLaw()
        relax_cfg = relax_cfg or RelaxConfig()
        stiff_cfg = stiff_cfg or StiffnessConfig()
        self._check(self._L.fibra_cuda_solve_device(
            self._ctx, C.c_void_p(F_dev_ptr), C.byref(law.c()), C.byref(relax_cfg.c()),
            C.byref(stiff_cfg.c()), int(want_tangent), C.c_void_p(out_dev_ptr)))

    def synchronize(self):
        self._check(self._L.fibra_cuda_synchronize(self._ctx))

    def last_stats(self) -> dict:
        s = _capi.SolveStats()
        self._check(self._L.fibra_cuda_last_stats(self._ctx, C.byref(s)))
        return {k: getattr(s, k) for k, _ in s._fields_}

    def fp64_peak(self) -> float:
        """Measured FP64-pipe lane-ops/s of this device (roofline denominator)."""
        v = C.c_double()
        self._check(self._L.fibra_cuda_fp64_peak(self._ctx, C.byref(v)))
        return v.value

    def close(self):
        if self._ctx:
            self._L.fibra_cuda_close(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_CTX_CACHE: Dict[tuple, DeviceBatch] = {}


def batch_response(library: RveLibrary, assignment: BatchAssignment, states: PackedStates,
                   law: FiberLaw, deformation, relax_cfg: RelaxConfig,
                   stiff_cfg: StiffnessConfig, pool=None, *, want_tangent: bool = True,
                   device: int = 0, devices: Optional[Sequence[int]] = None) -> BatchResult:
    """batch_response (batch.hpp:73-77, batch.cpp:155-187) on the B200.

    ``states`` is mutated in place exactly like the reference (warm start in, base solution
    out).  ``pool`` is accepted for signature parity and ignored: the GPU grid replaces
    the WorkerPool.  ``want_tangent=False`` runs the base solves only (sigma; C = 0).
    ``devices``: several GPUs of this process (DeviceBatch(devices=...)).
    """
    F = np.ascontiguousarray(deformation, dtype=np.float64).reshape(-1, 9)
    if len(F) != states.n_points():
        raise ConfigError("one deformation gradient per point is required")
    if len(assignment.entry_of_point) != states.n_points():
        raise ConfigError("assignment does not match the packed states")
    devs = tuple(int(d) for d in devices) if devices else (int(device),)
    # keyed on the library's entries (immutable networks), so an edited library re-uploads
    key = (id(library), tuple(id(e) for e in library.entries), devs,
           assignment.entry_of_point.tobytes())
    db = _CTX_CACHE.get(key)
    if db is None or db.library is not library:
        for k in list(_CTX_CACHE):
            if k[0] == id(library) and k[2] == devs:
                _CTX_CACHE.pop(k).close()
        db = DeviceBatch(library, assignment, devs[0], devices=devs)
        db.entries_ref = list(library.entries)  # keep the keyed entries alive
        _CTX_CACHE[key] = db
    tot = int(np.sum([library.entries[e].n_dof for e in assignment.entry_of_point]))
    n = db.n_points
    if (states.offsets.size != n + 1 or states.total_dofs() != tot
            or any(getattr(states, k).size != tot
                   for k in ("u", "v", "a", "f_int", "f_damp", "mass", "inv_mass"))
            or any(getattr(states, k).size != n for k in ("t", "iters", "converged"))):
        raise ConfigError("state layout does not match the network")  # relax.cpp:99-100
    db.upload_states(states)
    rec = db.solve(F, law, relax_cfg, stiff_cfg, want_tangent)
    db.download_states(states)
    return _to_result(rec)


@dataclass
class ProviderResult:  # macrofem.hpp:53-58
    responses: List[PointResponse]
    failed_points: List[int]
    microscale_iterations: int = 0
    solves_per_point: int = 0


class NetworkBatchProvider:
    """NetworkBatchProvider (batch.hpp:103-129): device-resident warm states across calls."""

    def __init__(self, region_of_point, library: RveLibrary, seed: int, law: FiberLaw = None,
                 relax_cfg: RelaxConfig = None, stiff_cfg: StiffnessConfig = None,
                 workers: int = 1, device: int = 0, devices: Optional[Sequence[int]] = None):
        self.library = library
        self.law = law or FiberLaw()
        self.relax_cfg = relax_cfg or RelaxConfig()
        self.stiff_cfg = stiff_cfg or StiffnessConfig()
        self._states, self.assignment = init_batch(region_of_point, library, seed)
        self._db = DeviceBatch(library, self.assignment, device, devices=devices)
        self._dirty = False
        self.total_solves = 0

    def states(self) -> PackedStates:
        if self._dirty:
            self._db.download_states(self._states)
            self._dirty = False
        return self._states

    def orientation(self, point: int, ref_dir) -> Optional[float]:
        """NetworkBatchProvider::orientation (batch.cpp:296-302): orientation_p2 of the
        point's current state; None when the point is out of range."""
        if point < 0 or point >= self._db.n_points:
            return None
        return float(self._db.orientation([point], ref_dir)[0])

    def respond(self, deformation) -> ProviderResult:
        rec = self._db.solve(deformation, self.law, self.relax_cfg, self.stiff_cfg, True)
        self._dirty = True
        # the next macro iteration revisits the same points: start the ones that relaxed
        # longest first (failed relaxations ran to the iteration cap)
        cost = np.where(rec["status"] == 0, rec["relax_iterations"].astype(np.float64),
                        np.where(np.isin(rec["status"], (6, 7)),
                                 7.0 * self.relax_cfg.max_iterations, 0.0))
        self._db.set_schedule(SCHED_HINT, cost)
        br = _to_result(rec)
        its = int(sum(s.relax_iterations for s in br.stats))
        self.total_solves += int(sum(s.solves for s in br.stats))
        return ProviderResult(br.responses, br.failed, its, br.stats[0].solves if br.stats else 0)
