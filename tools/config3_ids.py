"""Pick the config-3 golden sample: run the full 16,384-point config-3 batch on the GPU and
write every failed point plus 64 random converged ones (seed 1) to gpurun_out/config3_ids.txt.
The fixture itself is then computed from the reference build on the CPU:
  python tests/golden/make_golden_batches.py --only config3 --config3-ids config3_ids.txt"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2306_09427_b200 as P  # noqa: E402
from paper_2306_09427_b200 import synth  # noqa: E402

n = 16384
nets = synth.parallel_networks(synth.config3_network, range(n))
F = synth.batch_F(n).reshape(n, 9)
lib = P.RveLibrary(nets, policy="explicit", explicit_assignment=list(range(n)))
db = P.DeviceBatch(lib, P.BatchAssignment(np.arange(n, dtype=np.int32)))
rec = db.solve(F, want_tangent=False)
db.close()
failed = np.nonzero(rec["status"] != 0)[0]
ok = np.nonzero(rec["status"] == 0)[0]
pts = sorted(set(failed.tolist()) | set(np.random.default_rng(1).choice(ok, 64, replace=False).tolist()))
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "config3_ids.txt"), "w") as fh:
    fh.write("\n".join(map(str, pts)) + "\n")
print(f"{len(failed)} failed, status codes {np.unique(rec['status'][failed], return_counts=True)}; "
      f"wrote {len(pts)} ids")
