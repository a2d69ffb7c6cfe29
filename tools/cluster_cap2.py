"""Where cluster-path states differ from the oracle after a small cap."""
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
n = 32
pn, on = knn(712, 1900, 7)
nfree = pn.desc().n_free
F = batch_F(n)
lib = P.RveLibrary([pn])
for K in [int(a) for a in sys.argv[1:]]:
    st2 = O.PackedStates.fresh([on], [0] * n)
    O.batch_response([on], [0] * n, st2, F, relax_cfg=O.RelaxConfig(max_iterations=K),
                     want_tangent=False, n_threads=16)
    for rep in range(4):
        st, assign = P.init_batch(np.zeros(n, np.int32), lib, 0)
        P.batch_response(lib, assign, st, P.FiberLaw(), F, P.RelaxConfig(max_iterations=K),
                         P.StiffnessConfig(), want_tangent=False)
        nd = len(st.u) // n
        for p in range(n):
            sl = slice(p * nd, (p + 1) * nd)
            for key in ("u", "v", "f_int"):
                g, o = st.__dict__[key][sl] if key in st.__dict__ else getattr(st, key)[sl], st2.arrays[key][sl]
                d = np.nonzero(g.view(np.uint64) != o.view(np.uint64))[0]
                if len(d):
                    print(f"K={K} rep={rep} p={p} {key}: {len(d)} dofs differ (free<{nfree}): "
                          f"{d[:10].tolist()} max|diff| {np.abs(g[d]-o[d]).max():.3e} scale {np.abs(o).max():.3e}",
                          flush=True)
