"""Which records differ between two schedules (order-independence check)."""
import os
import sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_09427_b200 as P
from paper_2306_09427_b200.synth import batch_F, config1_spec

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
tangent = len(sys.argv) > 2
net = P.generate_network(config1_spec(), 1)
F = batch_F(n).reshape(n, 9)
db = P.DeviceBatch(P.RveLibrary([net]), P.BatchAssignment(np.zeros(n, np.int32)))
runs = []
for mode, hint in ((0, None), (1, None), (2, np.arange(n) % 7 + 1.0), (2, n - np.arange(n) + 0.0),
                   (0, None)):
    db.reset_states()
    db.set_schedule(mode, hint)
    runs.append(db.solve(F, want_tangent=tangent))
r0 = runs[0]
for i, r in enumerate(runs[1:], 1):
    bad = [p for p in range(n) if r[p].tobytes() != r0[p].tobytes()]
    print("run", i, "differs at", len(bad), "points", bad[:10])
    for p in bad[:3]:
        for k in r.dtype.names:
            if r[p][k].tobytes() != r0[p][k].tobytes():
                print("   p", p, k, r0[p][k], "->", r[p][k])
