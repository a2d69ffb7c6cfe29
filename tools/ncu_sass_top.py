"""Top SASS instructions by execution count from an ncu source CSV (cuda,sass)."""
import csv, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; cur = None; out = []; ops = Counter()
for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) != len(hdr): continue
    if r[0]:
        cur = r[0]; continue
    d = dict(zip(hdr, r))
    try:
        n = float(d.get("Instructions Executed", 0) or 0)
    except ValueError:
        continue
    sass = r[3].strip()
    op = sass.split()[0] if not sass.startswith("@") else sass.split()[1]
    ops[op.split(".")[0]] += n
    out.append((n, cur, r[2], sass[:70], d.get("Warp Stall Sampling (All Samples)", "0")))
tot = sum(o[0] for o in out)
print("by opcode:")
for op, n in ops.most_common(25):
    print(f"  {op:10s} {n/tot*100:5.1f}%")
if len(sys.argv) > 2:
    lo, hi = int(sys.argv[2]), int(sys.argv[3])
    for o in out:
        if o[1] and lo <= int(o[1]) <= hi:
            print(f"{o[0]:12.0f} {o[1]:>4} {o[2]} {o[3]:70s} {o[4]}")
