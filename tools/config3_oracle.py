"""Config-3 batch on the GPU vs the oracle on a sample: every failed point plus random
converged ones -- status, iterations and sigma bits."""
import os
import sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O
import paper_2306_09427_b200 as P
from paper_2306_09427_b200 import synth

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
n_ok = int(sys.argv[2]) if len(sys.argv) > 2 else 64
nets = synth.parallel_networks(synth.config3_network, range(n))
F = synth.batch_F(n).reshape(n, 9)
lib = P.RveLibrary(nets, policy="explicit", explicit_assignment=list(range(n)))
db = P.DeviceBatch(lib, P.BatchAssignment(np.arange(n, dtype=np.int32)))
rec = db.solve(F, want_tangent=False)
db.close()
failed = np.nonzero(rec["status"] != 0)[0]
ok = np.nonzero(rec["status"] == 0)[0]
pts = sorted(set(failed.tolist()) | set(np.random.default_rng(1).choice(ok, n_ok, replace=False).tolist()))
O.build(ref=False)
onets = [O.Network(nets[p].coords, nets[p].fiber_nodes[:, 0], nets[p].fiber_nodes[:, 1],
                   nets[p].fiber_area, nets[p].fiber_modulus, nets[p].box_half) for p in pts]
st = O.PackedStates.fresh(onets, list(range(len(pts))))
resp, status = O.batch_response(onets, list(range(len(pts))), st, F[pts].reshape(-1, 3, 3),
                                want_tangent=False, n_threads=os.cpu_count())
bad = 0
codes = {}
for i, p in enumerate(pts):
    g = rec[p]
    codes[int(status[i])] = codes.get(int(status[i]), 0) + 1
    same = int(g["status"]) == int(status[i])
    if same and not status[i]:
        o = resp[i]
        same = (int(g["base_report"]["iterations"]) == int(o["base_report"]["iterations"]) and
                g["sigma"].tobytes() == np.asarray(o["sigma"]).tobytes())
    if not same:
        bad += 1
        print("mismatch", p, int(g["status"]), int(status[i]), flush=True)
print(f"checked {len(pts)} points ({len(failed)} failed on the GPU), oracle status codes {codes}, "
      f"mismatching {bad}")
