"""Config-3 batch: default kernel selection vs all entries on 2-CTA clusters; report points
whose records differ (every path must be bit-identical) and check them on the oracle."""
import os
import sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O
import paper_2306_09427_b200 as P
from paper_2306_09427_b200 import synth

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
nets = synth.parallel_networks(synth.config3_network, range(n))
F = synth.batch_F(n).reshape(n, 9)
lib = P.RveLibrary(nets, policy="explicit", explicit_assignment=list(range(n)))
asg = P.BatchAssignment(np.arange(n, dtype=np.int32))
recs, shapes = [], []
for force in (None, "2"):
    if force:
        os.environ["FIBRA_FORCE_CLUSTER"] = force
    db = P.DeviceBatch(lib, asg)
    recs.append(db.solve(F, want_tangent=False))
    shapes.append([db.entry_kernel(i) for i in range(n)])
    db.close()
os.environ.pop("FIBRA_FORCE_CLUSTER", None)
a, b = recs
bad = [p for p in range(n) if a[p].tobytes() != b[p].tobytes()]
print("points", n, "differing", len(bad), "failed", int((a["status"] != 0).sum()), int((b["status"] != 0).sum()), flush=True)
O.build(ref=False)
for p in bad[:4]:
    net = nets[p]
    on = O.Network(net.coords, net.fiber_nodes[:, 0], net.fiber_nodes[:, 1], net.fiber_area,
                   net.fiber_modulus, net.box_half)
    st = O.PackedStates.fresh([on], [0])
    resp, status = O.batch_response([on], [0], st, F[p:p + 1], want_tangent=False)
    o = resp[0]
    def desc(r):
        return (int(r["status"]), int(r["base_report"]["iterations"]), r["sigma"][0])
    print(f"p={p} M={len(net.fiber_nodes)} N={len(net.coords)} default {shapes[0][p]} -> {desc(a[p])}; "
          f"cluster -> {desc(b[p])}; oracle -> {(int(status[0]), int(o['base_report']['iterations']), o['sigma'][0])}",
          flush=True)
