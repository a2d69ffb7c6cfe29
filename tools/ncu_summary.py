"""Curated metric table (metric,unit,value) of one ncu report, the same metric names as an
earlier summary: ncu_summary.py <report.ncu-rep> <reference_metrics.csv> <out.csv>."""
import csv
import subprocess
import sys

rep, ref, out = sys.argv[1:4]
names = [r[0] for r in list(csv.reader(open(ref)))[1:]]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
col = {h: i for i, h in enumerate(hdr)}
with open(out, "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(["metric", "unit", "value"])
    for n in names:
        if n in col:
            w.writerow([n, units[col[n]], vals[col[n]].replace(",", "")])
