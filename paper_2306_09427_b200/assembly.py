"""Macro assembly of the homogenized responses on the device.

Python mirror of the reference's macro-scale consumer of ``batch_response``:

* ``make_box_mesh``   -- macro_mesh.cpp:172-230 (structured box, 6-tet Kuhn cells, node sets)
* ``build_numbering`` -- macrofem.cpp:22-38 (free-first DOF numbering)
* ``assemble``        -- macrofem.cpp:104-187 (residual f_int - f_ext and the free x free
  material + geometric stiffness), computed by ``csrc/assembly.cu`` through the C-ABI
  ``fibra_cuda_assembly_*`` of ``include/fibra_cuda.h``; bit-identical to the reference.

``MacroAssembler`` holds the once-per-mesh plan (sparsity pattern and the element-to-slot
scatter) in HBM; ``assemble`` takes host arrays, ``assemble_device`` device pointers (for
example the result records a ``DeviceBatch.solve_device`` call left in HBM), so a Newton
iteration never copies the responses to the host.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _capi
from ._capi import ptr as _ptr

__all__ = ["MacroMesh", "DirichletBc", "DofNumbering", "Assembly", "MacroAssembler",
           "make_box_mesh", "build_numbering", "assemble"]

# Kuhn decomposition of a hex cell (macro_mesh.cpp:185-186)
_KTETS = ((0, 1, 3, 7), (0, 1, 7, 5), (0, 5, 7, 4), (0, 3, 2, 7), (0, 2, 6, 7), (0, 6, 4, 7))


@dataclass
class MacroMesh:  # macro_mesh.hpp
    ref_coords: np.ndarray            # (n_nodes, 3)
    coords: np.ndarray                # (n_nodes, 3) current
    tets: np.ndarray                  # (n_tets, 4) int32
    node_sets: Dict[str, np.ndarray] = field(default_factory=dict)

    @property
    def n_nodes(self) -> int:
        return len(self.ref_coords)

    @property
    def n_elements(self) -> int:
        return len(self.tets)

    @property
    def n_dof(self) -> int:
        return 3 * self.n_nodes


@dataclass
class DirichletBc:  # macro_mesh.hpp:46-53: a set value per axis (None = free) or affine
    node_set: str
    value: Sequence[Optional[float]] = (None, None, None)
    affine: Optional[np.ndarray] = None


@dataclass
class DofNumbering:  # macrofem.hpp:29-33
    n_free: int
    free_of_dof: np.ndarray   # int32, -1 where constrained
    constrained: np.ndarray   # uint8


def _vol6(a, b, c, d) -> float:  # tet_volume6 macro_mesh.cpp:14-21
    ab, ac, ad = b - a, c - a, d - a
    return (ab[0] * (ac[1] * ad[2] - ac[2] * ad[1]) - ab[1] * (ac[0] * ad[2] - ac[2] * ad[0]) +
            ab[2] * (ac[0] * ad[1] - ac[1] * ad[0]))


def make_box_mesh(nx: int, ny: int, nz: int, lx: float = 1.0, ly: float = 1.0,
                  lz: float = 1.0) -> MacroMesh:
    """make_box_mesh (macro_mesh.cpp:172-230): (nx+1)(ny+1)(nz+1) nodes, 6 tets per cell,
    positively oriented, face node sets xmin..zmax."""
    if nx < 1 or ny < 1 or nz < 1:
        raise ValueError("box mesh needs >= 1 cell per axis")
    k, j, i = np.meshgrid(np.arange(nz + 1), np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
    ref = np.stack([lx * i.ravel() / nx, ly * j.ravel() / ny, lz * k.ravel() / nz], axis=1)

    def nid(ii, jj, kk):
        return (kk * (ny + 1) + jj) * (nx + 1) + ii

    kc, jc, ic = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    ic, jc, kc = ic.ravel(), jc.ravel(), kc.ravel()
    corners = np.stack([nid(ic, jc, kc), nid(ic + 1, jc, kc), nid(ic, jc + 1, kc),
                        nid(ic + 1, jc + 1, kc), nid(ic, jc, kc + 1), nid(ic + 1, jc, kc + 1),
                        nid(ic, jc + 1, kc + 1), nid(ic + 1, jc + 1, kc + 1)], axis=1)
    tets = corners[:, np.array(_KTETS)].reshape(-1, 4).astype(np.int32)
    x = ref[tets]
    ab, ac, ad = x[:, 1] - x[:, 0], x[:, 2] - x[:, 0], x[:, 3] - x[:, 0]
    v6 = np.einsum("ij,ij->i", ab, np.cross(ac, ad))
    neg = v6 < 0
    tets[neg, 2], tets[neg, 3] = tets[neg, 3].copy(), tets[neg, 2].copy()
    ii, jj, kk = i.ravel(), j.ravel(), k.ravel()
    sets = {"xmin": np.nonzero(ii == 0)[0], "xmax": np.nonzero(ii == nx)[0],
            "ymin": np.nonzero(jj == 0)[0], "ymax": np.nonzero(jj == ny)[0],
            "zmin": np.nonzero(kk == 0)[0], "zmax": np.nonzero(kk == nz)[0]}
    sets = {n: s.astype(np.int32) for n, s in sets.items()}
    return MacroMesh(ref, ref.copy(), tets, sets)


def build_numbering(mesh: MacroMesh, dirichlet: Sequence[DirichletBc] = ()) -> DofNumbering:
    """build_numbering (macrofem.cpp:22-38): constrained axes of every Dirichlet set, then
    free slots in DOF order."""
    constrained = np.zeros(mesh.n_dof, np.uint8)
    for bc in dirichlet:
        nodes = np.asarray(mesh.node_sets[bc.node_set], dtype=np.int64)
        for k in range(3):
            if bc.affine is not None or bc.value[k] is not None:
                constrained[3 * nodes + k] = 1
    free = constrained == 0
    fod = np.full(mesh.n_dof, -1, np.int32)
    fod[free] = np.arange(int(free.sum()), dtype=np.int32)
    return DofNumbering(int(free.sum()), fod, constrained)


@dataclass
class Assembly:  # macrofem.hpp:72-75
    residual: np.ndarray      # (n_free,) f_int - f_ext
    col_ptr: np.ndarray       # (n_free+1,) int64  -- Eigen compressed column-major storage
    row_idx: np.ndarray       # (nnz,) int32, ascending within each column
    values: np.ndarray        # (nnz,)

    @property
    def stiffness(self):
        import scipy.sparse as sp
        n = len(self.residual)
        return sp.csc_matrix((self.values, self.row_idx, self.col_ptr), shape=(n, n))


def _check(as_handle, rc: int, bad: Optional[int] = None):
    if rc == 0:
        return
    from . import _raise
    L = _capi.load(build_if_missing=False)
    msg = L.fibra_cuda_assembly_last_error(as_handle) if as_handle else b""
    msg = msg.decode() if msg else ""
    where = f" (element {bad})" if bad is not None and bad >= 0 else ""
    _raise(rc, f"assemble: {msg or _capi.STATUS_NAMES.get(rc, rc)}{where}")


class MacroAssembler:
    """The once-per-mesh assembly plan on one device (fibra_cuda_assembly_create)."""

    def __init__(self, mesh: MacroMesh, numbering: DofNumbering, device: int = 0):
        self._L = _capi.load()
        self.mesh, self.numbering = mesh, numbering
        tets = np.ascontiguousarray(mesh.tets, dtype=np.int32)
        fod = np.ascontiguousarray(numbering.free_of_dof, dtype=np.int32)
        h = C.c_void_p()
        rc = self._L.fibra_cuda_assembly_create(device, _ptr(tets, _capi._ip), len(tets),
                                                mesh.n_nodes, _ptr(fod, _capi._ip),
                                                numbering.n_free, C.byref(h))
        _check(None, rc)
        self._h = h
        nnz = C.c_int64(0)
        self._L.fibra_cuda_assembly_pattern(h, C.byref(nnz), None, None)
        self.nnz = nnz.value
        self.col_ptr = np.zeros(numbering.n_free + 1, np.int64)
        self.row_idx = np.zeros(self.nnz, np.int32)
        self._L.fibra_cuda_assembly_pattern(h, None, _ptr(self.col_ptr, _capi._lp),
                                            _ptr(self.row_idx, _capi._ip))

    def info(self) -> dict:
        out = np.zeros(5, np.int64)
        self._L.fibra_cuda_assembly_info(self._h, _ptr(out, _capi._lp))
        return dict(zip(("n_tets", "n_nodes", "n_free", "nnz", "node_pairs"), out.tolist()))

    def set_stream(self, cuda_stream: int):
        _check(self._h, self._L.fibra_cuda_assembly_set_stream(self._h, C.c_void_p(cuda_stream)))

    def assemble(self, coords, sigma=None, spatial_c=None, f_ext_free=None, responses=None,
                 stride: int = 42, out=None) -> Assembly:
        """Host arrays in and out.  Responses either as ``sigma`` (n,6) + ``spatial_c``
        (n,6,6), or as ``responses``: a float64 record array whose rows start with the 42
        doubles of a PointResponse (``stride`` doubles per row).  ``out`` = optional
        (residual[n_free], values[nnz]) float64 buffers (e.g. pinned) to write into."""
        n = self.mesh.n_elements
        if responses is None:
            responses = np.empty((n, 42))
            responses[:, :6] = np.asarray(sigma, dtype=np.float64).reshape(n, 6)
            responses[:, 6:] = np.asarray(spatial_c, dtype=np.float64).reshape(n, 36)
            stride = 42
        responses = np.asarray(responses)
        if responses.dtype.names is not None:  # record array (e.g. RESULT_DTYPE): raw bytes
            if responses.dtype.itemsize % 8:
                raise ValueError("response records must be a whole number of doubles")
            resp = np.ascontiguousarray(responses).view(np.float64).reshape(-1)
        else:  # numeric input is converted, never reinterpreted
            resp = np.ascontiguousarray(responses, dtype=np.float64).reshape(-1)
        if stride < 42 or resp.size < stride * n:
            raise ValueError(f"responses hold {resp.size} doubles, {n} elements x stride "
                             f"{stride} (>= 42) needed")
        x = np.ascontiguousarray(coords, dtype=np.float64)
        if x.size != 3 * self.mesh.n_nodes:
            raise ValueError(f"coords must be ({self.mesh.n_nodes}, 3)")
        x = x.reshape(-1)
        fe = None if f_ext_free is None else np.ascontiguousarray(f_ext_free, dtype=np.float64)
        if fe is not None and fe.size != self.numbering.n_free:
            raise ValueError(f"f_ext_free must have n_free = {self.numbering.n_free} entries")
        if out is None:
            res, vals = np.zeros(self.numbering.n_free), np.zeros(self.nnz)
        else:
            res, vals = out
            if (res.dtype != np.float64 or vals.dtype != np.float64 or not res.flags.c_contiguous
                    or not vals.flags.c_contiguous or res.size != self.numbering.n_free
                    or vals.size != self.nnz):
                raise ValueError("out must be contiguous float64 (n_free,) and (nnz,) arrays")
        bad = C.c_int32(-1)
        rc = self._L.fibra_cuda_assemble(self._h, _ptr(x, _capi._dp), _ptr(resp, _capi._dp),
                                         stride, None if fe is None else _ptr(fe, _capi._dp),
                                         _ptr(res, _capi._dp), _ptr(vals, _capi._dp),
                                         C.byref(bad))
        _check(self._h, rc, bad.value)
        return Assembly(res, self.col_ptr, self.row_idx, vals)

    def assemble_device(self, coords_ptr: int, responses_ptr: int, stride: int,
                        f_ext_ptr: Optional[int], residual_ptr: int, values_ptr: int):
        """Device pointers; asynchronous on the assembler's stream (``status`` syncs)."""
        rc = self._L.fibra_cuda_assemble_device(self._h, C.c_void_p(coords_ptr),
                                                C.c_void_p(responses_ptr), stride,
                                                C.c_void_p(f_ext_ptr) if f_ext_ptr else None,
                                                C.c_void_p(residual_ptr), C.c_void_p(values_ptr))
        _check(self._h, rc)

    def status(self):
        bad = C.c_int32(-1)
        rc = self._L.fibra_cuda_assembly_status(self._h, C.byref(bad))
        _check(self._h, rc, bad.value)

    def times_ms(self) -> List[float]:
        ms = (C.c_float * 3)()
        _check(self._h, self._L.fibra_cuda_assembly_times(self._h, ms))
        return list(ms)

    def close(self):
        if getattr(self, "_h", None):
            self._L.fibra_cuda_assembly_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def assemble(mesh: MacroMesh, numbering: DofNumbering, responses, f_ext_free=None,
             device: int = 0) -> Assembly:
    """assemble (macrofem.cpp:104-187) for a list of PointResponse (``.sigma`` (6,),
    ``.spatial_c`` (6,6)).  One-shot: plans the pattern, assembles, frees the plan."""
    if len(responses) != mesh.n_elements:
        from . import ConfigError
        raise ConfigError("one response per element is required")
    sig = np.array([np.asarray(r.sigma, dtype=np.float64) for r in responses]).reshape(-1, 6)
    cm = np.array([np.asarray(r.spatial_c, dtype=np.float64) for r in responses]).reshape(-1, 36)
    asm = MacroAssembler(mesh, numbering, device)
    try:
        return asm.assemble(mesh.coords, sig, cm, f_ext_free)
    finally:
        asm.close()
