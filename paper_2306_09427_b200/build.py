"""Build the in-tree CUDA library ``paper_2306_09427_b200/lib/libfibra_b200.so``.

sm_100a only (``-gencode arch=compute_100a,code=sm_100a``).  ``--fmad=false`` is part of
the numerical contract: the reference forbids FMA contraction (proj/CMakeLists.txt:14-16)
and the DR trajectory is reproduced bit for bit.  Host C++ gets ``-ffp-contract=off`` for
the same reason (the network generator must emit the reference's exact coordinates).

``FIBRA_PHASE_PROF=1`` builds the diagnostics variant ``libfibra_b200_prof.so`` whose DR
kernel accumulates per-warp phase cycle counters (see dr_kernel.cuh FB_PROF); the loader
picks it when the same variable is set at run time.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_DIR = os.path.join(HERE, "lib")
PROF = bool(os.environ.get("FIBRA_PHASE_PROF"))
LIB = os.path.join(LIB_DIR, "libfibra_b200_prof.so" if PROF else "libfibra_b200.so")
# diagnostics: FIBRA_LIB=<path> loads a prebuilt layout-experiment library (tools/variants.py)
# as is, without the staleness rebuild
LIB_OVERRIDE = os.environ.get("FIBRA_LIB")
if LIB_OVERRIDE:
    LIB = LIB_OVERRIDE
SOURCES = [
    os.path.join(HERE, "csrc", "fibra_cuda.cu"),
    os.path.join(HERE, "csrc", "kernels_resident.cu"),
    os.path.join(HERE, "csrc", "kernels_cluster.cu"),
    os.path.join(HERE, "csrc", "kernels_node.cu"),
    os.path.join(HERE, "csrc", "kernels_stream.cu"),
    os.path.join(HERE, "csrc", "assembly.cu"),
    os.path.join(HERE, "csrc", "host", "network.cpp"),
    os.path.join(HERE, "csrc", "host", "netgen.cpp"),
    os.path.join(HERE, "csrc", "host", "schedule.cpp"),
    os.path.join(HERE, "csrc", "host", "cluster_schedule.cpp"),
    os.path.join(HERE, "csrc", "host", "node_schedule.cpp"),
]
DEPS = SOURCES + [
    os.path.join(HERE, "csrc", "dr_kernel.cuh"),
    os.path.join(HERE, "csrc", "dr_cluster.cuh"),
    os.path.join(HERE, "csrc", "dr_node.cuh"),
    os.path.join(HERE, "csrc", "dr_stream.cuh"),
    os.path.join(HERE, "csrc", "host", "node_schedule.hpp"),
    os.path.join(HERE, "csrc", "variants.hpp"),
    os.path.join(HERE, "csrc", "host", "cluster_schedule.hpp"),
    os.path.join(HERE, "csrc", "tensor.cuh"),
    os.path.join(HERE, "csrc", "fastmath.cuh"),
    os.path.join(HERE, "csrc", "host", "host_internal.hpp"),
    os.path.join(HERE, "csrc", "host", "schedule.hpp"),
    os.path.join(ROOT, "include", "fibra_cuda.h"),
]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every translation unit to an object (in parallel), then link the library."""
    if LIB_OVERRIDE:
        return LIB
    if not force and not _stale():
        return LIB
    os.makedirs(LIB_DIR, exist_ok=True)
    obj_dir = os.path.join(LIB_DIR, "obj_prof" if PROF else "obj")
    os.makedirs(obj_dir, exist_ok=True)
    flags = ["-O3", "-std=c++17", *ARCH, "--fmad=false", "-lineinfo",
             "-Xptxas", "-v" if verbose else "-O3",
             "-Xcompiler", "-fPIC,-ffp-contract=off,-O3",
             "-I", os.path.join(ROOT, "include"), "-I", os.path.join(HERE, "csrc"),
             *(["-DFIBRA_PHASE_PROF=1"] if PROF else [])]
    objs = [os.path.join(obj_dir, os.path.basename(src) + ".o") for src in SOURCES]

    def compile_one(args):
        src, obj = args
        return subprocess.run([NVCC, *flags, "-c", "-o", obj, src], capture_output=True, text=True)

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(compile_one, zip(SOURCES, objs)))
    for r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc build of libfibra_b200.so failed")
        if verbose:
            sys.stderr.write(r.stderr)
    r = subprocess.run([NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-ldl"],
                       capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link of libfibra_b200.so failed")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
