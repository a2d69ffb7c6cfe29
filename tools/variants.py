"""Build layout-experiment variants of the resident DR kernel (diagnostics).

Each variant recompiles csrc/kernels_resident.cu with extra -D flags and links it with the
product objects into paper_2306_09427_b200/lib/variants/<name>.so (and <name>_prof.so with
FIBRA_PHASE_PROF); run one with FIBRA_LIB=<path>.  usage: variants.py name=FLAGS ...
e.g. variants.py topo0="-DFIBRA_TOPO_REG=0" vnode="-DFIBRA_VERDICT_NODE=1"
"""
import os
import shlex
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_09427_b200 import build as B  # noqa: E402

B.build()
out_dir = os.path.join(B.LIB_DIR, "variants")
os.makedirs(out_dir, exist_ok=True)
obj_dir = os.path.join(B.LIB_DIR, "obj")
res_src = os.path.join(B.HERE, "csrc", "kernels_resident.cu")
flags = ["-O3", "-std=c++17", *B.ARCH, "--fmad=false", "-lineinfo", "-Xptxas", "-O3",
         "-Xcompiler", "-fPIC,-ffp-contract=off,-O3", "-I", os.path.join(B.ROOT, "include"),
         "-I", os.path.join(B.HERE, "csrc")]
others = [os.path.join(obj_dir, os.path.basename(s) + ".o") for s in B.SOURCES if s != res_src]
jobs = []
for arg in sys.argv[1:]:
    name, _, extra = arg.partition("=")
    for prof in (False, True):
        nm = name + ("_prof" if prof else "")
        jobs.append((nm, shlex.split(extra) + (["-DFIBRA_PHASE_PROF=1"] if prof else [])))


def one(job):
    nm, extra = job
    obj = os.path.join(out_dir, nm + ".o")
    r = subprocess.run([B.NVCC, *flags, *extra, "-c", "-o", obj, res_src], capture_output=True,
                       text=True)
    if r.returncode:
        return nm, r.stderr[-2000:]
    r = subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", os.path.join(out_dir, nm + ".so"), obj,
                        *others, "-ldl"], capture_output=True, text=True)
    os.remove(obj)
    return nm, r.stderr[-2000:] if r.returncode else "ok"


with ThreadPoolExecutor(max_workers=4) as ex:
    for nm, msg in ex.map(one, jobs):
        print(nm, msg)
