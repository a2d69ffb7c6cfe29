"""Repeat the schedule test case and report which records differ (diagnostics)."""
import os
import sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2306_09427_b200 as P
from _pairs import batch_F, knn

a = knn(14, 38, 101, neighbors=9)
b = knn(12, 32, 102, neighbors=9)
lib = P.RveLibrary([a[0], b[0]])
n = 40
F = batch_F(n)
F[5] = np.diag([1e-9, 1e-9, 1e-9])
F[17] = np.diag([-1.0, 1.0, 1.0])
F[23] = np.eye(3)
runs = []
for mode in (0, 0, 0, 1, 1, 1):
    st, assign = P.init_batch(np.zeros(n, np.int32), lib, 3)
    db = P.DeviceBatch(lib, assign)
    db.set_schedule(mode)
    runs.append((mode, db.solve(F, want_tangent=True)))
    db.close()
r0 = runs[0][1]
print("entries", assign.entry_of_point[:12])
for i, (mode, r) in enumerate(runs[1:], 1):
    bad = [p for p in range(n) if r[p].tobytes() != r0[p].tobytes()]
    print("run", i, "mode", mode, "differs at", bad)
    for p in bad[:4]:
        fields = [k for k in r.dtype.names if r[p][k].tobytes() != r0[p][k].tobytes()]
        print("   p", p, fields, "its", r0[p]["relax_iterations"], r[p]["relax_iterations"],
              "status", r0[p]["status"], r[p]["status"])
