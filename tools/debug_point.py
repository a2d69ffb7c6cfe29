"""One config-3 point on the GPU vs the oracle after a small iteration cap: which DOFs differ."""
import os
import sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O
import paper_2306_09427_b200 as P
from paper_2306_09427_b200 import synth

p = int(sys.argv[1])  # env FIBRA_FORCE_CLUSTER / FIBRA_CLUSTER_MIRROR select the kernel path
net = synth.config3_network(p)
F = synth.batch_F(p + 1)[p:p + 1]
on = O.Network(net.coords, net.fiber_nodes[:, 0], net.fiber_nodes[:, 1], net.fiber_area,
               net.fiber_modulus, net.box_half)
O.build(ref=False)
lib = P.RveLibrary([net])
for cap in [int(a) for a in sys.argv[2:]] or [1, 2, 10]:
    st, asg = P.init_batch(np.zeros(1, np.int32), lib, 0)
    db = P.DeviceBatch(lib, asg)
    shape = db.entry_kernel(0)
    rec = db.solve(F, relax_cfg=P.RelaxConfig(max_iterations=cap), want_tangent=False)
    db.download_states(st)
    db.close()
    ost = O.PackedStates.fresh([on], [0])
    resp, status = O.batch_response([on], [0], ost, F, relax_cfg=O.RelaxConfig(max_iterations=cap),
                                    want_tangent=False)
    print(f"cap {cap}: shape {shape} gpu status {rec['status'][0]} oracle {status[0]}")
    for k in ("u", "f_int", "v"):
        g, o = getattr(st, k), ost.arrays[k]
        d = np.nonzero(g.view(np.uint64) != o.view(np.uint64))[0]
        print(f"   {k}: {len(d)} dofs differ; first {d[:12].tolist()} nonfinite gpu {int((~np.isfinite(g)).sum())}")
