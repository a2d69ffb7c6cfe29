"""CPU: csrc/libm_glibc.cuh -- the exponential fibre law's expm1 / exp restated from the host
libm's FMA builds (glibc 2.39) -- equals the host libm bit for bit (compiled here as host
code with -ffp-contract=off, explicit fma() where the library fuses)."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = r"""
#include "libm_glibc.cuh"
extern "C" void run(int which, const double* x, long long n, double* out) {
  for (long long i = 0; i < n; ++i)
    out[i] = which ? fibra_b200::glibc::expm1(x[i]) : fibra_b200::glibc::exp(x[i]);
}
"""


@pytest.fixture(scope="module")
def restated(tmp_path_factory):
    d = tmp_path_factory.mktemp("libm")
    (d / "r.cpp").write_text(SRC)
    so = d / "r.so"
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-shared", "-fPIC",
                    "-I", os.path.join(ROOT, "paper_2306_09427_b200", "csrc"), "-o", str(so),
                    str(d / "r.cpp")], check=True)
    L = C.CDLL(str(so))
    L.run.argtypes = [C.c_int, C.POINTER(C.c_double), C.c_longlong, C.POINTER(C.c_double)]
    return L


def operands(seed):
    rng = np.random.default_rng(seed)
    parts = [rng.uniform(lo, hi, 1_000_000) for lo, hi in
             ((-1, 1), (-0.35, 0.35), (-1.1, 1.1), (-5, 5), (-60, 60), (-700, 700))]
    parts.append(rng.choice([-1, 1], 200_000) * 10.0 ** rng.uniform(-300, 0, 200_000))
    parts.append(np.array([0.0, -0.0, 1e-310, -1e-310, 0.5 * np.log(2), np.log(2), 1.5 * np.log(2),
                           56 * np.log(2), 709.78, -745.0, np.inf, -np.inf, np.nan]))
    return np.concatenate(parts)


@pytest.mark.parametrize("which", [0, 1])
def test_restatement_equals_host_libm(oracle_lib, restated, which):
    import oracle as O
    x = operands(17 + which)
    want = O.libm(which, x)
    got = np.empty_like(x)
    dp = C.POINTER(C.c_double)
    restated.run(which, x.ctypes.data_as(dp), x.size, got.ctypes.data_as(dp))
    same = (got.view(np.uint64) == want.view(np.uint64)) | (np.isnan(got) & np.isnan(want))
    assert same.all(), x[~same][:5]
