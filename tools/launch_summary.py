"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV).

usage: python tools/launch_summary.py launches.csv [last_n]
last_n: only the last N launches (the timed steps of the bench command)."""
import csv
import sys
from collections import defaultdict

lines = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
hdr = rows[0]
iN, iV, iM = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
recs = [(r[iN], float(r[iV].replace(",", ""))) for r in rows[1:] if len(r) > iV and r[iM] == "gpu__time_duration.sum"]
if len(sys.argv) > 2:
    recs = recs[-int(sys.argv[2]):]
agg = defaultdict(list)
for n, v in recs:
    agg[n.split("(")[0][:60]].append(v)
tot = sum(sum(v) for v in agg.values())
print(f"{len(recs)} launches, {tot/1000:.1f} us total device time")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:60s} n={len(v):5d} mean={sum(v)/len(v)/1000:9.2f} us  share={sum(v)/tot:6.1%}")
