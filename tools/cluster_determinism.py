"""Cluster path determinism: the same stress-only batch twice on the GPU and once on the oracle."""
import os
import sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O
import paper_2306_09427_b200 as P
from _pairs import batch_F, knn, same_bits

O.build()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 48
pn, on = knn(712, 1900, 7)
F = batch_F(n)
lib = P.RveLibrary([pn])
db = P.DeviceBatch(lib, P.BatchAssignment(np.zeros(n, np.int32)))
print("kernel", db.entry_kernel(0))
runs = []
for rep in range(3):
    db.reset_states()
    runs.append(db.solve(F, want_tangent=False))
st = O.PackedStates.fresh([on], [0] * n)
resp, status = O.batch_response([on], [0] * n, st, F, want_tangent=False, n_threads=16)
for rep, r in enumerate(runs):
    bad = [p for p in range(n) if r[p]["base_report"]["iterations"] != resp[p]["base_report"]["iterations"]
           or not same_bits(r[p]["sigma"], resp[p]["sigma"])]
    print("run", rep, "mismatching points", bad[:20],
          [(int(runs[rep][p]["base_report"]["iterations"]), int(resp[p]["base_report"]["iterations"])) for p in bad[:5]])
