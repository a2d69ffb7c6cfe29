import sys, numpy as np, torch
sys.path.insert(0,'.')
import paper_2306_09427_b200 as P
from paper_2306_09427_b200 import _capi
print(torch.cuda.get_device_properties(0))
net = P.generate_lattice_network(23, 50000, 1)
for sh in range(4):
    out = np.zeros(4, np.int64)
    _capi.load().fibra_debug_cluster_smem(net.desc(), 16, sh, out.ctypes.data_as(_capi._lp))
    print(sh, out)
try:
    db = P.DeviceBatch(P.RveLibrary([net]), P.BatchAssignment(np.zeros(1, np.int32)))
    print(db.entry_kernel(0))
except Exception as e:
    print("ERR", e)
