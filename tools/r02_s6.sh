#!/bin/bash
# item-size A/B on small steps + ncu source capture of the fp32 decode kernel at C1
mkdir -p gpurun_out
for cfg in "2 64" "1 64" "1 128" "0.5 128" "0 256"; do
  set -- $cfg
  echo "items_per_warp=$1 min_rows=$2" >> gpurun_out/s6_ab.log
  HGCA_ITEMS_PER_WARP=$1 HGCA_MIN_ITEM_ROWS=$2 timeout 300 python tools/fixed_cost_probe.py C1 C5S >> gpurun_out/s6_ab.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" -k regex:decode_f32 -s 20 -c 1 \
    -o gpurun_out/s6_f32 python tools/fixed_cost_probe.py C1 > gpurun_out/s6_ncu_log.txt 2>&1
python tools/ncu_summary.py gpurun_out/s6_f32.ncu-rep 40 > gpurun_out/s6_f32_summary.txt 2>&1
cat gpurun_out/s6_ab.log; head -60 gpurun_out/s6_f32_summary.txt
