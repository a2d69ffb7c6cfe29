"""ctypes binding of the C-ABI declared in include/fibra_cuda.h.

The library is the in-tree ``paper_2306_09427_b200/lib/libfibra_b200.so`` (built by
``build.py``).  There is no fallback: if it is missing or no sm_100 device is present the
calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os

from . import build as _build

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)
_bp = C.POINTER(C.c_uint8)

FIBRA_OK = 0
STATUS_NAMES = {0: "ok", 1: "config", 2: "kinematics", 3: "collapse", 4: "bad_dt",
                5: "diverged", 6: "not_converged", 7: "probe_failed", 8: "singular",
                10: "non-finite stress response", 11: "non-finite assembled residual",
                20: "cuda", 21: "arg", 22: "io"}

# every symbol include/fibra_cuda.h declares (checked by tests/test_capi.py)
EXPORTS = [
    "fibra_network_create", "fibra_network_generate", "fibra_network_generate_lattice",
    "fibra_network_read",
    "fibra_network_write", "fibra_network_describe", "fibra_network_free",
    "fibra_host_last_error", "fibra_assign_random", "fibra_schedule_report",
    "fibra_cluster_report", "fibra_schedule_slots", "fibra_debug_cluster_forces",
    "fibra_debug_resident_forces", "fibra_debug_cluster_smem", "fibra_debug_node_forces",
    "fibra_cuda_open", "fibra_cuda_open_devices", "fibra_plan_shards", "fibra_network_cost",
    "fibra_cuda_close", "fibra_cuda_last_error", "fibra_cuda_set_stream",
    "fibra_cuda_upload_library", "fibra_cuda_bind_points", "fibra_cuda_reset_states",
    "fibra_cuda_set_schedule", "fibra_cuda_entry_kernel", "fibra_cuda_orientation",
    "fibra_cuda_upload_states", "fibra_cuda_download_states", "fibra_cuda_solve",
    "fibra_cuda_solve_device", "fibra_cuda_synchronize", "fibra_cuda_last_stats",
    "fibra_cuda_device_count", "fibra_cuda_fp64_peak", "fibra_cuda_phase_profile", "fibra_cuda_trace",
    "fibra_cuda_selftest_fastmath", "fibra_cuda_eval_libm",
    "fibra_cuda_assembly_create", "fibra_cuda_assembly_set_stream", "fibra_cuda_assembly_pattern",
    "fibra_cuda_assemble", "fibra_cuda_assemble_device", "fibra_cuda_assembly_status",
    "fibra_cuda_assembly_times", "fibra_cuda_assembly_info", "fibra_cuda_assembly_last_error",
    "fibra_cuda_assembly_free",
]


class NetgenSpec(C.Structure):
    _fields_ = [("style", C.c_int32), ("fibers", C.c_int32), ("nodes", C.c_int32),
                ("half_length", C.c_double), ("merge_radius", C.c_double),
                ("neighbors", C.c_int32), ("align_bias", C.c_double),
                ("align_axis", C.c_double * 3), ("fiber_area", C.c_double),
                ("fiber_modulus", C.c_double), ("box_half", C.c_double),
                ("tol_bnd", C.c_double)]


class NetDesc(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("n_fibers", C.c_int32), ("n_free", C.c_int32),
                ("n_boundary", C.c_int32), ("coords", _dp), ("fiber_nodes", _ip),
                ("fiber_area", _dp), ("fiber_modulus", _dp), ("packed_of_dof", _ip),
                ("packed_ref", _dp), ("fiber_packed_dofs", _ip), ("rest_length", _dp),
                ("node_lump", _dp), ("boundary_nodes", _ip), ("box_half", C.c_double),
                ("max_ea", C.c_double)]


class Law(C.Structure):
    _fields_ = [("kind", C.c_int32), ("ea_scale", C.c_double), ("nonlinearity", C.c_double),
                ("buckling_off", C.c_int32)]


class RelaxCfg(C.Structure):
    _fields_ = [("damping", C.c_double), ("tolerance", C.c_double),
                ("max_iterations", C.c_int64), ("dt_safety", C.c_double),
                ("density_scale", C.c_double), ("energy_check", C.c_int32)]


class StiffCfg(C.Structure):
    _fields_ = [("fd_rel_step", C.c_double), ("reuse_warm", C.c_int32)]


class RelaxReport(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("residual", C.c_double), ("eps_eff", C.c_double),
                ("kinetic_fraction", C.c_double), ("dt", C.c_double),
                ("converged", C.c_int32), ("reserved0", C.c_int32),
                ("energy_drift", C.c_double)]


class PointResult(C.Structure):
    _fields_ = [("sigma", C.c_double * 6), ("spatial_c", C.c_double * 36),
                ("pk2", C.c_double * 6), ("material_a", C.c_double * 36),
                ("stress_asymmetry", C.c_double), ("base_report", RelaxReport),
                ("solves", C.c_int32), ("reserved1", C.c_int32), ("relax_iterations", C.c_int64),
                ("failed_probe", C.c_int32), ("status", C.c_int32)]


class SolveStats(C.Structure):
    _fields_ = [("solves", C.c_int64), ("iterations", C.c_int64),
                ("fiber_iterations", C.c_int64), ("pipe_ops", C.c_int64),
                ("dr_kernel_ms", C.c_float), ("total_ms", C.c_float),
                ("kernel_launches", C.c_int32), ("alg_flops", C.c_int64)]


_lib = None


def lib_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True):
    """Load libfibra_b200.so (building it in-tree with nvcc when stale or absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_missing:
        _build.build()
    if not os.path.exists(_build.LIB):
        raise RuntimeError(f"CUDA library missing: {_build.LIB} (run python -m "
                           "paper_2306_09427_b200.build); there is no CPU fallback")
    L = C.CDLL(_build.LIB)
    vp = C.c_void_p
    pp = C.POINTER(C.c_void_p)
    sig = {
        "fibra_network_create": (C.c_int, [_dp, C.c_int32, _ip, _dp, _dp, C.c_int32, C.c_double,
                                           C.c_double, pp]),
        "fibra_network_generate": (C.c_int, [C.POINTER(NetgenSpec), C.c_uint64, pp]),
        "fibra_network_read": (C.c_int, [C.c_char_p, C.c_double, C.c_double, pp]),
        "fibra_network_generate_lattice": (C.c_int, [C.c_int32, C.c_int32, C.c_double, C.c_double,
                                                     C.c_double, C.c_double, C.c_double,
                                                     C.c_uint64, pp]),
        "fibra_network_write": (C.c_int, [vp, C.c_char_p]),
        "fibra_network_describe": (C.c_int, [vp, C.POINTER(NetDesc)]),
        "fibra_network_free": (None, [vp]),
        "fibra_host_last_error": (C.c_char_p, []),
        "fibra_assign_random": (C.c_int, [C.c_uint64, C.c_int32, C.c_int32, _ip]),
        "fibra_schedule_report": (C.c_int, [C.POINTER(NetDesc), C.c_int, C.c_int, C.c_int, _lp]),
        "fibra_cluster_report": (C.c_int, [C.POINTER(NetDesc), C.c_int, C.c_int, C.c_int, C.c_int,
                                           _lp]),
        "fibra_debug_cluster_forces": (C.c_int, [C.POINTER(NetDesc), C.c_int, C.c_int, C.c_int,
                                                 _dp, _dp, _dp]),
        "fibra_debug_cluster_smem": (C.c_int, [C.POINTER(NetDesc), C.c_int, C.c_int, _lp]),
        "fibra_debug_resident_forces": (C.c_int, [C.POINTER(NetDesc), C.c_int, _dp, _dp, _dp]),
        "fibra_debug_node_forces": (C.c_int, [C.POINTER(NetDesc), C.c_int, _dp, _dp, _lp]),
        "fibra_schedule_slots": (C.c_int, [C.POINTER(NetDesc), C.c_int, C.c_int, C.c_int, _ip,
                                           C.c_int32]),
        "fibra_cuda_open": (C.c_int, [C.c_int, pp]),
        "fibra_cuda_eval_libm": (C.c_int, [vp, C.c_int32, _dp, C.c_int64, _dp]),
        "fibra_cuda_open_devices": (C.c_int, [_ip, C.c_int32, pp]),
        "fibra_plan_shards": (C.c_int, [_dp, C.c_int32, C.c_int32, _ip]),
        "fibra_network_cost": (C.c_int, [C.POINTER(NetDesc), _dp]),
        "fibra_cuda_close": (C.c_int, [vp]),
        "fibra_cuda_last_error": (C.c_char_p, [vp]),
        "fibra_cuda_set_stream": (C.c_int, [vp, vp]),
        "fibra_cuda_upload_library": (C.c_int, [vp, C.POINTER(NetDesc), C.c_int32]),
        "fibra_cuda_bind_points": (C.c_int, [vp, _ip, C.c_int32]),
        "fibra_cuda_reset_states": (C.c_int, [vp]),
        "fibra_cuda_set_schedule": (C.c_int, [vp, C.c_int32, _dp]),
        "fibra_cuda_entry_kernel": (C.c_int, [vp, C.c_int32, _ip]),
        "fibra_cuda_orientation": (C.c_int, [vp, _ip, C.c_int32, _dp, _dp]),
        "fibra_cuda_upload_states": (C.c_int, [vp, _dp, _dp, _lp, _bp]),
        "fibra_cuda_download_states": (C.c_int, [vp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                                 _lp, _bp]),
        "fibra_cuda_solve": (C.c_int, [vp, _dp, C.POINTER(Law), C.POINTER(RelaxCfg),
                                       C.POINTER(StiffCfg), C.c_int32, C.POINTER(PointResult)]),
        "fibra_cuda_solve_device": (C.c_int, [vp, vp, C.POINTER(Law), C.POINTER(RelaxCfg),
                                              C.POINTER(StiffCfg), C.c_int32, vp]),
        "fibra_cuda_synchronize": (C.c_int, [vp]),
        "fibra_cuda_last_stats": (C.c_int, [vp, C.POINTER(SolveStats)]),
        "fibra_cuda_device_count": (C.c_int, [C.POINTER(C.c_int)]),
        "fibra_cuda_fp64_peak": (C.c_int, [vp, C.POINTER(C.c_double)]),
        "fibra_cuda_selftest_fastmath": (C.c_int, [vp, C.c_uint64, C.c_uint64,
                                                   C.POINTER(C.c_uint64)]),
        "fibra_cuda_trace": (C.c_int, [vp, C.POINTER(C.c_uint64), C.c_size_t,
                                       C.POINTER(C.c_size_t)]),
        "fibra_cuda_phase_profile": (C.c_int, [vp, C.POINTER(C.c_uint64), C.c_size_t,
                                               C.POINTER(C.c_size_t)]),
        "fibra_cuda_assembly_create": (C.c_int, [C.c_int, _ip, C.c_int32, C.c_int32, _ip,
                                                 C.c_int32, pp]),
        "fibra_cuda_assembly_set_stream": (C.c_int, [vp, vp]),
        "fibra_cuda_assembly_pattern": (C.c_int, [vp, _lp, _lp, _ip]),
        "fibra_cuda_assemble": (C.c_int, [vp, _dp, _dp, C.c_int64, _dp, _dp, _dp, _ip]),
        "fibra_cuda_assemble_device": (C.c_int, [vp, vp, vp, C.c_int64, vp, vp, vp]),
        "fibra_cuda_assembly_status": (C.c_int, [vp, _ip]),
        "fibra_cuda_assembly_times": (C.c_int, [vp, C.POINTER(C.c_float)]),
        "fibra_cuda_assembly_info": (C.c_int, [vp, _lp]),
        "fibra_cuda_assembly_last_error": (C.c_char_p, [vp]),
        "fibra_cuda_assembly_free": (C.c_int, [vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def ptr(a, t):
    return a.ctypes.data_as(t)
