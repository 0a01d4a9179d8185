#!/bin/bash
# round-2 session 3: where the small-step fixed cost goes (device kernel durations, timelines)
mkdir -p gpurun_out
tag=s8
timeout 300 python tools/fixed_cost_probe.py > gpurun_out/${tag}_probe.log 2>&1
timeout 600 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_launch.csv python tools/fixed_cost_probe.py EMPTY EMPTYB C1 C1B C5S > gpurun_out/${tag}_launch_run.log 2>&1
python - <<'PY' > gpurun_out/${tag}_launch_summary.txt 2>&1
import csv
lines=open("gpurun_out/s8_launch.csv").read().splitlines()
st=[i for i,l in enumerate(lines) if l.startswith('"ID"')][0]
rows=list(csv.reader(lines[st:])); h=rows[0]
iN,iV,iM=h.index("Kernel Name"),h.index("Metric Value"),h.index("Metric Name")
recs=[(r[iN].split("(")[0][:40],float(r[iV].replace(",",""))) for r in rows[1:] if len(r)>iV and r[iM]=="gpu__time_duration.sum"]
# 5 configs x 200 timed steps x 2 kernels (+maintenance); print per block of 400 decode/merge launches
import collections
blk=collections.OrderedDict(); cur=0; n=0
for name,v in recs:
    blk.setdefault(cur,collections.defaultdict(list))[name].append(v/1000)
    if name.startswith("void decode_merge"):
        n+=1
        if n%200==0: cur+=1
for c,d in blk.items():
    print("config", ["EMPTY","EMPTYB","C1","C1B","C5S"][c] if c<5 else c)
    for k,v in d.items():
        v=sorted(v); print(f"   {k:40s} n={len(v):4d} p50={v[len(v)//2]:8.2f} min={v[0]:8.2f} max={v[-1]:8.2f} us")
PY
for c in EMPTY C1; do timeout 300 python tools/timeline_f32.py $c > gpurun_out/${tag}_tl_$c.log 2>&1; done
HGCA_TL_CFG=C5S timeout 300 python tools/timeline.py > gpurun_out/${tag}_tl_c5s.log 2>&1
cat gpurun_out/${tag}_probe.log gpurun_out/${tag}_launch_summary.txt
tail -6 gpurun_out/${tag}_tl_EMPTY.log; tail -6 gpurun_out/${tag}_tl_C1.log; tail -12 gpurun_out/${tag}_tl_c5s.log
