"""Print the bank-aware schedule quality (host only, no GPU)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_09427_b200 as P  # noqa: E402
from paper_2306_09427_b200 import _capi  # noqa: E402

spec = P.NetGenSpec(style="knn", nodes=375, fibers=1000, neighbors=10)
for seed in (1, 2, 4):
    net = P.generate_network(spec, seed)
    out = np.zeros(7, np.int64)
    for T, FPT, NPT in ((384, 3, 1), (512, 4, 1)):
        _capi.load().fibra_schedule_report(C.byref(net.desc()), T, FPT, NPT,
                                           out.ctypes.data_as(_capi._lp))
        print(f"seed {seed} T={T} FPT={FPT}: fits={out[0]} conflicting_groups={out[1]} "
              f"gather_excess={out[2]} steps={out[3]} ({out[2]/max(out[3],1):.2f}/step) "
              f"store_excess={out[6]} gd_slots={out[4]} node_slots={out[5]}")
