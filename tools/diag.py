import time, numpy as np, sys
sys.path.insert(0, "/root/repo")
import paper_2306_09427_b200 as P
from paper_2306_09427_b200.synth import batch_F, config1_spec
net = P.generate_network(config1_spec(), 1)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
F = batch_F(n).reshape(n, 9)
lib = P.RveLibrary([net]); assign = P.BatchAssignment(np.zeros(n, np.int32))
db = P.DeviceBatch(lib, assign)
print("fp64 peak Gop/s", db.fp64_peak()/1e9)
for tang in (False,):
    db.reset_states()
    t = time.perf_counter(); rec = db.solve(F, want_tangent=tang); dt = time.perf_counter() - t
    s = db.last_stats()
    it = rec["base_report"]["iterations"]
    print("tangent", tang, "wall", dt, s)
    print("iters min/mean/max", it.min(), it.mean(), it.max(), "failed", (rec["status"]!=0).sum(), np.bincount(rec["status"]))
    print("us per RVE-iter per SM:", s["dr_kernel_ms"]*1e3*148/s["iterations"])
    print("pipe frac", s["pipe_ops"]/(s["dr_kernel_ms"]*1e-3)/db.fp64_peak())
