"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum
--csv --log-file X.csv):  python tools/launch_summary.py X.csv "header line" """
import collections
import csv
import re
import sys

S = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
idx = {k: i for i, k in enumerate(rows[0])}
agg = collections.defaultdict(lambda: [0.0, 0])
for r in rows[1:]:
    if r[idx["Metric Name"]] != "gpu__time_duration.sum":
        continue
    v = float(r[idx["Metric Value"]].replace(",", "")) * S[r[idx["Metric Unit"]]]
    m = re.match(r"(void )?([\w:<>, ]+?)\(", r[idx["Kernel Name"]])
    k = m.group(2) if m else r[idx["Kernel Name"]]
    agg[k][0] += v
    agg[k][1] += 1
tot = sum(a[0] for a in agg.values())
if len(sys.argv) > 2:
    print(sys.argv[2])
for k, (t, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{t:10.3f} ms {100 * t / tot:5.1f}%  x{n:<4d} {k}  ({t / n:.3f} ms each)")
print(f"total {tot:.1f} ms over {sum(a[1] for a in agg.values())} launches")
