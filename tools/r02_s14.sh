#!/bin/bash
mkdir -p gpurun_out
tag=s14
for c in EMPTYB C5S; do HGCA_TL_CFG=$c timeout 300 python tools/timeline.py > gpurun_out/${tag}_tl_$c.log 2>&1; done
timeout 300 python tools/timeline_f32.py C1 > gpurun_out/${tag}_tl_C1.log 2>&1
timeout 600 ncu --nvtx --nvtx-include "timed_graph/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_launch.csv python tools/fixed_cost_probe.py EMPTYB > gpurun_out/${tag}_launch_run.log 2>&1
python tools/launch_summary.py gpurun_out/${tag}_launch.csv > gpurun_out/${tag}_launch_summary.txt 2>&1
for c in EMPTYB C5S; do tail -12 gpurun_out/${tag}_tl_$c.log; done; tail -8 gpurun_out/${tag}_tl_C1.log; cat gpurun_out/${tag}_launch_summary.txt
