"""Config-2 DR kernel time under each base-solve schedule (results must be identical)."""
import os
import sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_09427_b200 as P
from paper_2306_09427_b200.synth import batch_F, config1_spec

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
tangent = len(sys.argv) > 2 and sys.argv[2] == "tangent"
net = P.generate_network(config1_spec(), 1)
F = batch_F(n).reshape(n, 9)
db = P.DeviceBatch(P.RveLibrary([net]), P.BatchAssignment(np.zeros(n, np.int32)))
ref = None
for mode in (P.SCHED_BATCH, P.SCHED_STRAIN, P.SCHED_HINT):
    db.reset_states()
    if mode == P.SCHED_HINT:
        cost = np.where(ref["status"] == 0, ref["relax_iterations"], 5e5 * 7).astype(float)
        db.set_schedule(mode, cost)
    else:
        db.set_schedule(mode)
    rec = db.solve(F, want_tangent=tangent)
    s = db.last_stats()
    same = ref is None or rec.tobytes() == ref.tobytes()
    ref = rec if ref is None else ref
    print(f"mode {mode}: dr_kernel {s['dr_kernel_ms']:.1f} ms total {s['total_ms']:.1f} ms "
          f"iters {s['iterations']} identical={same}", flush=True)
