"""Sum ncu per-line instruction counts and stall samples into phases
(line ranges of solve.cu given as name=lo-hi) plus per-file totals.
    python tools/ncu_phases.py source.csv name=lo-hi ..."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
ranges = []
for a in sys.argv[2:]:
    name, r = a.split("=")
    lo, hi = r.split("-")
    ranges.append((name, int(lo), int(hi)))
agg = defaultdict(lambda: [0.0, 0.0])
fname, cur, hdr = "", None, None
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
        cur = (fname, int(r[0]))
    if cur is None:
        continue
    try:
        s, ins = float(r[4] or 0), float(r[7] or 0)
    except ValueError:
        continue
    key = cur[0]
    if cur[0] == "solve.cu":
        for name, lo, hi in ranges:
            if lo <= cur[1] <= hi:
                key = name
                break
    agg[key][0] += s
    agg[key][1] += ins
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:24s} instr {v[1] / 1e6:9.1f}M ({100 * v[1] / ti:5.1f}%)  stall-samples {100 * v[0] / ts:5.1f}%")
