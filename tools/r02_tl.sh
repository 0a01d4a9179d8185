#!/bin/bash
# per-warp timelines (debug build) of small steps + the fixed-cost probe at HEAD
mkdir -p gpurun_out
tag=${1:-tl}
for c in EMPTYB C5S C2; do HGCA_TL_CFG=$c timeout 300 python tools/timeline.py > gpurun_out/${tag}_tl_$c.log 2>&1; done
for c in C1 EMPTY; do timeout 300 python tools/timeline_f32.py $c > gpurun_out/${tag}_tl_$c.log 2>&1; done
timeout 600 python tools/fixed_cost_probe.py > gpurun_out/${tag}_probe.log 2>&1
for c in EMPTYB C5S C2 C1 EMPTY; do echo "== $c"; tail -14 gpurun_out/${tag}_tl_$c.log; done; cat gpurun_out/${tag}_probe.log
