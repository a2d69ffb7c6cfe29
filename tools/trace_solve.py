"""Per-solve timeline of one batch (FIBRA_TRACE): occupancy over time and the tail.

usage: trace_solve.py config2|config3|config5 [n]
"""
import ctypes as C
import os
import sys
import numpy as np
os.environ["FIBRA_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_09427_b200 as P
from paper_2306_09427_b200 import _capi, synth

which = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else {"config2": 1024, "config3": 16384, "config5": 4096}[which]
tangent = which == "config5"
if which == "config2":
    nets = [P.generate_network(synth.config1_spec(), 1)]
    eop = np.zeros(n, np.int32)
else:
    nets = synth.parallel_networks(synth.config3_network, range(n))
    eop = np.arange(n, dtype=np.int32)
F = synth.batch_F(n).reshape(n, 9)
lib = P.RveLibrary(nets, policy="explicit", explicit_assignment=list(eop)) if which != "config2" else P.RveLibrary(nets)
db = P.DeviceBatch(lib, P.BatchAssignment(eop))
for rep in range(2):
    db.reset_states()
    rec = db.solve(F, want_tangent=tangent)
L = _capi.load()
nn = C.c_size_t(0)
L.fibra_cuda_trace(db._ctx, None, 0, C.byref(nn))
buf = (C.c_uint64 * nn.value)()
L.fibra_cuda_trace(db._ctx, buf, nn.value, C.byref(nn))
tr = np.frombuffer(buf, np.uint64).reshape(-1, 4).astype(np.int64)
os.makedirs("gpurun_out", exist_ok=True)
np.save(f"gpurun_out/trace_{which}.npy", tr)
np.save(f"gpurun_out/status_{which}.npy", rec["status"])
ran = tr[:, 0] > 0
t0 = tr[ran, 0].min()
st, en = (tr[:, 0] - t0) / 1e6, (tr[:, 1] - t0) / 1e6
span = en[ran].max()
busy = (en - st)[ran].sum()
slots = len(set((tr[ran, 2]).tolist()))
print(f"{which} n={n}: solves run {ran.sum()} on {slots} CTAs, span {span:.0f} ms, "
      f"busy {busy / (slots * span):.1%} of CTA-time")
base = np.arange(len(tr)) < n
print(f"  bases: last start {st[base & ran].max():.0f} ms, last end {en[base & ran].max():.0f} ms; "
      f"probes: first start {st[~base & ran].min() if (~base & ran).any() else 0:.0f} ms")
edges = np.linspace(0, span, 21)
occ = []
for a, b in zip(edges[:-1], edges[1:]):
    ov = np.clip(np.minimum(en[ran], b) - np.maximum(st[ran], a), 0, None).sum()
    occ.append(ov / (slots * (b - a)))
print("  occupancy per 5% of the span:", " ".join(f"{o:.2f}" for o in occ))
d = (en - st)[ran]
its = tr[ran, 3]
print(f"  solve ms: median {np.median(d):.2f}, p99 {np.percentile(d, 99):.1f}, max {d.max():.1f}; "
      f"iterations median {np.median(its):.0f}, max {its.max()}")
cls = (tr[:, 2] >> 24) & 0xff
for k in sorted(set(cls[ran].tolist())):
    m = ran & (cls == k)
    print(f"  class {k}: solves {m.sum()}, start {st[m].min():.0f} ms, end {en[m].max():.0f} ms, "
          f"longest {np.max(en[m] - st[m]):.0f} ms (starts {st[m][np.argmax(en[m] - st[m])]:.0f}), "
          f"CTA-busy {(en[m] - st[m]).sum():.0f} ms, CTAs {len(set(tr[m, 2].tolist()))}")
late = np.argsort(-en)[:5]
for s in late:
    kind = "base" if s < n else f"probe {(s - n) % 6} of {(s - n) // 6}"
    print(f"  late: solve {s} ({kind}) class {cls[s]} {st[s]:.0f}-{en[s]:.0f} ms, iterations {tr[s, 3]}")
