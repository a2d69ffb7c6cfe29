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
