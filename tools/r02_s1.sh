#!/bin/bash
# round-2 GPU session 1: state check + fixed-cost probe (run under gpurun)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s1_smi.txt 2>&1
lscpu | head -20 > gpurun_out/s1_lscpu.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/s1_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/s1_tests.log
timeout 300 python bench.py --no-cpu-baseline --steps 200 > gpurun_out/s1_bench.log 2>&1
timeout 300 python tools/fixed_cost_probe.py > gpurun_out/s1_probe.log 2>&1
timeout 600 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/s1_launch.csv python tools/fixed_cost_probe.py EMPTY C1 C5S > gpurun_out/s1_launch_run.log 2>&1
python tools/launch_summary.py gpurun_out/s1_launch.csv > gpurun_out/s1_launch_summary.txt 2>&1
tail -3 gpurun_out/s1_tests.log; cat gpurun_out/s1_probe.log; cat gpurun_out/s1_launch_summary.txt; tail -1 gpurun_out/s1_bench.log | cut -c1-600
