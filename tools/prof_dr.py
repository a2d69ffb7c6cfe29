"""Profiling driver: one DR launch on the config-1 network (148 points, fixed iteration cap)."""
import sys
import os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_09427_b200 as P
from paper_2306_09427_b200.synth import batch_F, config1_spec

n = int(sys.argv[1]) if len(sys.argv) > 1 else 148
its = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
net = P.generate_network(config1_spec(), 1)
F = batch_F(n).reshape(n, 9)
db = P.DeviceBatch(P.RveLibrary([net]), P.BatchAssignment(np.zeros(n, np.int32)))
cfg = P.RelaxConfig(max_iterations=its)
db.solve(F, relax_cfg=cfg, want_tangent=False)
db.reset_states()
rec = db.solve(F, relax_cfg=cfg, want_tangent=False)
s = db.last_stats()
print(s, "us/iter/CTA:", s["dr_kernel_ms"] * 1e3 / its)
if os.environ.get("FIBRA_PHASE_PROF"):
    import ctypes as C
    from paper_2306_09427_b200 import _capi
    L = _capi.load()
    nn = C.c_size_t()
    L.fibra_cuda_phase_profile(db._ctx, None, 0, C.byref(nn))
    buf = (C.c_uint64 * nn.value)()
    L.fibra_cuda_phase_profile(db._ctx, buf, nn.value, C.byref(nn))
    a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 8).astype(float)[:, :6] / its
    nw = a.shape[0] // (len(F) if len(F) < 296 else 296)
    print("per-iteration cycles per warp (mean over CTAs): fiber, bar1, node checks, gather, "
          "update+decider, bar2")
    a = a.reshape(-1, nw, 6)
    for w in range(nw):
        print(w, np.round(a[:, w].mean(0), 1))
