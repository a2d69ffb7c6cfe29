"""Host emulation of one force pass from the uploaded entry arrays (resident and cluster
kernels), bitwise against direct per-fiber assembly, over config-3 networks and every shape
that fits: catches plan/upload bugs without a GPU (fibra_debug_*_forces)."""
import os
import sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2306_09427_b200 import _capi, synth


def check(net, u):
    lib, dp = _capi.load(), _capi._dp
    d = net.desc()
    n = u.size
    bad = []
    for sh in range(8):  # shapes past the table return FIBRA_E_ARG (21)
        fe, fd = np.zeros(n), np.zeros(n)
        r = lib.fibra_debug_resident_forces(d, sh, u.ctypes.data_as(dp), fe.ctypes.data_as(dp),
                                            fd.ctypes.data_as(dp))
        if r == 0 and (fe.view(np.uint64) != fd.view(np.uint64)).any() or r not in (0, 1, 21):
            bad.append(("resident", sh, r))
    for C in (2, 4):
        for sh in range(3):
            for mirror in (1, 0):
                fe, fd = np.zeros(n), np.zeros(n)
                r = lib.fibra_debug_cluster_forces(d, C, sh, mirror, u.ctypes.data_as(dp),
                                                   fe.ctypes.data_as(dp), fd.ctypes.data_as(dp))
                if r == 0 and (fe.view(np.uint64) != fd.view(np.uint64)).any() or r not in (0, 1):
                    bad.append(("cluster", C, sh, mirror, r))
    return bad


if __name__ == "__main__":
    lo, hi = int(sys.argv[1]), int(sys.argv[2])
    for p in range(lo, hi):
        net = synth.config3_network(p)
        u = np.random.default_rng(p).normal(0, 0.01, net.packed_ref_coords.size)
        b = check(net, u)
        if b:
            print(p, len(net.fiber_nodes), b, flush=True)
