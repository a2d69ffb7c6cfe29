"""Cluster-path tangent diagnostics: relax_iterations and tangent vs the oracle."""
import os
import sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O
import paper_2306_09427_b200 as P
from _pairs import batch_F, knn, oracle_batch, same_bits

O.build()
pn, on = knn(712, 1900, 7)
sp, so = knn(14, 38, 101, neighbors=9)
for label, nets, onets, eop in (("cluster-only", [pn], [on], [0, 0]),
                                ("mixed", [sp, pn], [so, on], [1, 0, 1, 0])):
    F = batch_F(len(eop))
    lib = P.RveLibrary(nets, policy="explicit", explicit_assignment=eop)
    st, assign = P.init_batch(np.zeros(len(eop), np.int32), lib, 0)
    for reuse in (1, 0):
        sc = P.StiffnessConfig(reuse_warm=bool(reuse))
        br = P.batch_response(lib, assign, st, P.FiberLaw(), F, P.RelaxConfig(), sc)
        st2 = O.PackedStates.fresh(onets, eop)
        resp, status = O.batch_response(onets, eop, st2, F, reuse_warm=bool(reuse),
                                        want_tangent=True, n_threads=8)
        for p in range(len(eop)):
            r = br.records[p]
            print(label, "reuse", reuse, "p", p, "entry", eop[p], "its gpu/oracle",
                  r["relax_iterations"], resp[p]["relax_iterations"],
                  "base", r["base_report"]["iterations"], resp[p]["base_report"]["iterations"],
                  "C same", same_bits(r["spatial_c"].reshape(6, 6), resp[p]["spatial_c"]), flush=True)
        st, assign = P.init_batch(np.zeros(len(eop), np.int32), lib, 0)
