import csv
import sys
from collections import defaultdict

lines = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
hdr = rows[0]
iN, iV = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = defaultdict(list)
for r in rows[1:]:
    if len(r) > iV:
        agg[r[iN][:70]].append(float(r[iV].replace(",", "")))
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:70s} n={len(v):4d} mean={sum(v)/len(v)/1000:9.2f}us share={sum(v)/tot:6.1%}")
