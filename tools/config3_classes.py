"""Config-3 batch (or the config-5 tangent batch: `n tangent`) on one GPU: per kernel class
points and completion time (FIBRA_CLASS_TIMES)."""
import os
import sys
import numpy as np
os.environ["FIBRA_CLASS_TIMES"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_09427_b200 as P
from paper_2306_09427_b200 import synth

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
tangent = len(sys.argv) > 2 and sys.argv[2] == "tangent"
nets = synth.parallel_networks(synth.config3_network, range(n))
F = synth.batch_F(n).reshape(n, 9)
db = P.DeviceBatch(P.RveLibrary(nets, policy="explicit", explicit_assignment=list(range(n))),
                   P.BatchAssignment(np.arange(n, dtype=np.int32)))
for rep in range(2):
    db.reset_states()
    rec = db.solve(F, want_tangent=tangent)
    s = db.last_stats()
    print(f"rep {rep}: dr {s['dr_kernel_ms']:.0f} ms, iterations {s['iterations']:.3g}, failed {(rec['status'] != 0).sum()}", flush=True)
