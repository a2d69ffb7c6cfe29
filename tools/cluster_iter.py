"""Per-iteration time of one DR solve on the resident vs cluster kernels (fixed cap)."""
import os
import sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_09427_b200 as P
from paper_2306_09427_b200.synth import batch_F, config1_spec

which = sys.argv[1]
n = int(sys.argv[2])
its = int(sys.argv[3]) if len(sys.argv) > 3 else 4000
if which == "config1":
    net = P.generate_network(config1_spec(), 1)
elif which == "knn1900":
    net = P.generate_network(P.NetGenSpec(style="knn", nodes=712, fibers=1900, neighbors=10), 7)
elif which == "knn5k":
    net = P.generate_network(P.NetGenSpec(style="knn", nodes=1250, fibers=5000, neighbors=10), 3)
else:
    net = P.generate_lattice_network(23, 50000, 1)
F = batch_F(n).reshape(n, 9)
db = P.DeviceBatch(P.RveLibrary([net]), P.BatchAssignment(np.zeros(n, np.int32)))
cfg = P.RelaxConfig(max_iterations=its, tolerance=1e-30)
db.solve(F, relax_cfg=cfg, want_tangent=False)
db.reset_states()
db.solve(F, relax_cfg=cfg, want_tangent=False)
s = db.last_stats()
print(f"{which} n={n} kernel={db.entry_kernel(0)} force={os.environ.get('FIBRA_FORCE_CLUSTER')} "
      f"iters={s['iterations']} dr_ms={s['dr_kernel_ms']:.2f} us/iter/solve={s['dr_kernel_ms']*1e3/its:.3f} "
      f"RVE-iter/s={s['iterations']/(s['dr_kernel_ms']*1e-3):.3e}")
