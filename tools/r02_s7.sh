#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/s7_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/s7_tests.log
for cfg in "2 64" "1 64" "1 128" "0.5 128" "0 256"; do
  set -- $cfg
  echo "items_per_warp=$1 min_rows=$2" >> gpurun_out/s7_ab.log
  HGCA_ITEMS_PER_WARP=$1 HGCA_MIN_ITEM_ROWS=$2 timeout 300 python tools/fixed_cost_probe.py C1 C5S >> gpurun_out/s7_ab.log 2>&1
done
timeout 300 python tools/timeline_f32.py C1 > gpurun_out/s7_tl_c1.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/s7_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" -k regex:decode_f32 -s 20 -c 1 \
    -o gpurun_out/s7_f32 python tools/fixed_cost_probe.py C1 > gpurun_out/s7_ncu_log.txt 2>&1
python tools/ncu_summary.py gpurun_out/s7_f32.ncu-rep 30 > gpurun_out/s7_f32_summary.txt 2>&1
tail -3 gpurun_out/s7_tests.log; cat gpurun_out/s7_ab.log; tail -7 gpurun_out/s7_tl_c1.log; tail -1 gpurun_out/s7_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C3', d['value'], d['ms_per_step'], d['roofline']['frac'], 'C2', d['c2']['value'], d['c2']['roofline_frac'])"
head -45 gpurun_out/s7_f32_summary.txt
