"""Aggregate an ncu 'source' page (cuda,sass CSV) per CUDA source line."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = defaultdict(lambda: defaultdict(float))
src = {}
cur = None
for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    if r[0]:
        cur = int(r[0])
        src[cur] = r[1][:90]
        continue
    d = dict(zip(hdr, r))
    for k in ("Warp Stall Sampling (All Samples)", "Instructions Executed",
              "L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal", "stall_barrier",
              "stall_short_sb", "stall_long_sb", "stall_math", "stall_mio", "stall_wait",
              "stall_lg", "stall_not_selected", "stall_selected", "stall_branch_resolving",
              "stall_dispatch", "stall_no_inst"):
        try:
            agg[cur][k] += float(d.get(k, 0) or 0)
        except ValueError:
            pass
tot = sum(v["Warp Stall Sampling (All Samples)"] for v in agg.values())
toti = sum(v["Instructions Executed"] for v in agg.values())
print(f"total samples {tot:.0f} instructions {toti:.3g}")
keys = ["stall_barrier", "stall_short_sb", "stall_long_sb", "stall_math", "stall_mio",
        "stall_wait", "stall_lg", "stall_not_selected", "stall_selected", "stall_branch_resolving",
        "stall_dispatch", "stall_no_inst"]
top = sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]
for line, v in top:
    s = v["Warp Stall Sampling (All Samples)"]
    st = ", ".join(f"{k[6:]}={v[k]/max(s,1)*100:.0f}%" for k in keys if v[k] / max(s, 1) > 0.08)
    print(f"{line:4d} {s/tot*100:5.1f}% inst {v['Instructions Executed']/toti*100:5.1f}% "
          f"wf {v['L1 Wavefronts Shared']:.3g}/{v['L1 Wavefronts Shared Ideal']:.3g} | {src.get(line,'')} | {st}")
