"""Per-CUDA-line totals from an ncu 'source' page (cuda,sass CSV), normalised per unit.

usage: ncu_lines2.py <csv> <units> [min_instr_per_unit]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
N = float(sys.argv[2])
lim = float(sys.argv[3]) if len(sys.argv) > 3 else 8
hdr = None
fname = "?"
agg = defaultdict(lambda: [0.0, 0.0, 0.0])
src = {}
cur = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        src[cur] = r[1][:80]
        continue
    d = dict(zip(hdr, r))

    def f(k):
        try:
            return float(d.get(k, 0) or 0)
        except ValueError:
            return 0.0
    a = agg[cur]
    a[0] += f("Instructions Executed") / N
    a[1] += f("Warp Stall Sampling (All Samples)")
    a[2] += f("L1 Wavefronts Shared") / N
tots = sum(v[1] for v in agg.values()) or 1
tot_i = sum(v[0] for v in agg.values())
print(f"total instructions/unit {tot_i:.1f}")
for k in sorted(k for k in agg if k):
    v = agg[k]
    if v[0] >= lim or v[1] / tots > 0.004:
        print(f"{k[0][:10]:>10}:{k[1]:<4} {v[0]:7.1f} st={v[1]/tots*100:5.1f}% wf={v[2]:6.1f}  {src.get(k, '')}")
