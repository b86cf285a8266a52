"""Aggregate an ncu source page (cuda,sass CSV) by CUDA source line.
    ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > s.csv
    python tools/ncu_lines.py s.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = defaultdict(lambda: [0.0, 0.0, ""])
fname = ""
cur = None
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 8:
        continue
    if r[0]:
        cur = (fname, r[0], r[1].strip()[:90])
    if cur is None:
        continue
    try:
        s = float(r[4] or 0)
        ins = float(r[7] or 0)
    except ValueError:
        continue
    a = agg[cur]
    a[0] += s
    a[1] += ins
tot = sum(v[0] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * v[0] / tot:5.1f}%  {v[1]:12.0f}  {k[0]}:{k[1]:>4}  {k[2]}")
