#!/bin/bash
# ncu --set full + source of the fp32 decode and its merge at C1 (eager steps)
mkdir -p gpurun_out
tag=s11
for k in decode_f32 decode_merge; do
  timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" -k regex:${k} -s 20 -c 1 \
    -o gpurun_out/${tag}_${k} python tools/fixed_cost_probe.py C1 > gpurun_out/${tag}_${k}_log.txt 2>&1
  python tools/ncu_summary.py gpurun_out/${tag}_${k}.ncu-rep 40 > gpurun_out/${tag}_${k}_summary.txt 2>&1
  head -60 gpurun_out/${tag}_${k}_summary.txt
done
