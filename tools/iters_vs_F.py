"""Dump per-point iteration counts of config 2 with their F (for scheduling heuristics)."""
import os
import sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_09427_b200 as P
from paper_2306_09427_b200.synth import batch_F, config1_spec

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
net = P.generate_network(config1_spec(), 1)
F = batch_F(n).reshape(n, 9)
db = P.DeviceBatch(P.RveLibrary([net]), P.BatchAssignment(np.zeros(n, np.int32)))
rec = db.solve(F, want_tangent=False)
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/iters_config2.npz", F=F, iters=rec["base_report"]["iterations"], status=rec["status"])
print("saved", rec["base_report"]["iterations"][:10])
