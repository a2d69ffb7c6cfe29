"""Cluster path vs oracle: full PackedStates after an iteration cap K (trajectory parity)."""
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
F = batch_F(n)
lib = P.RveLibrary([pn])
for K in [int(a) for a in sys.argv[1:]] or [20, 200, 2000, 20000]:
    st2 = O.PackedStates.fresh([on], [0] * n)
    resp, status = O.batch_response([on], [0] * n, st2, F, relax_cfg=O.RelaxConfig(max_iterations=K),
                                    want_tangent=False, n_threads=16)
    off = st2.arrays["offsets"] if "offsets" in st2.arrays else None
    for rep in range(2):
        st, assign = P.init_batch(np.zeros(n, np.int32), lib, 0)
        br = P.batch_response(lib, assign, st, P.FiberLaw(), F, P.RelaxConfig(max_iterations=K),
                              P.StiffnessConfig(), want_tangent=False)
        nd = len(st.u) // n
        bad = [p for p in range(n) if not same_bits(st.u[p * nd:(p + 1) * nd], st2.arrays["u"][p * nd:(p + 1) * nd])]
        bad_it = [p for p in range(n) if st.iters[p] != st2.arrays["iters"][p]]
        print(f"K={K} rep={rep} u mismatch {len(bad)} {bad[:8]} iters mismatch {len(bad_it)} "
              f"status gpu {np.bincount(br.records['status'], minlength=8)[:8]} oracle {np.bincount(status, minlength=8)[:8]}",
              flush=True)
