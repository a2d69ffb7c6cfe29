"""Exponential law: GPU vs oracle deviation (libm vs CUDA expm1/exp), resident and cluster."""
import os
import sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O
import paper_2306_09427_b200 as P
from _pairs import batch_F, knn

O.build()
for label, args in (("resident", (375, 1000, 1)), ("cluster", (712, 1900, 7))):
    pn, on = knn(*args)
    n = 6
    F = batch_F(n)
    for B in (1.2, 4.0):
        lib = P.RveLibrary([pn])
        st, assign = P.init_batch(np.zeros(n, np.int32), lib, 0)
        br = P.batch_response(lib, assign, st, P.FiberLaw(kind="exponential", nonlinearity=B), F,
                              P.RelaxConfig(), P.StiffnessConfig(), want_tangent=True)
        st2 = O.PackedStates.fresh([on], [0] * n)
        resp, status = O.batch_response([on], [0] * n, st2, F, law=O.Law(kind=1, nonlinearity=B),
                                        want_tangent=True, n_threads=16)
        for p in range(n):
            r = br.records[p]
            ds = np.abs(r["sigma"] - resp[p]["sigma"]).max() / np.abs(resp[p]["sigma"]).max()
            dc = np.abs(r["spatial_c"].reshape(6, 6) - resp[p]["spatial_c"]).max() / np.abs(resp[p]["spatial_c"]).max()
            print(f"{label} B={B} p={p} status {r['status']}/{status[p]} its {r['base_report']['iterations']}/"
                  f"{resp[p]['base_report']['iterations']} rel dsigma {ds:.2e} rel dC {dc:.2e}", flush=True)
