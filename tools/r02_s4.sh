#!/bin/bash
mkdir -p gpurun_out
./tools/bin/probe_dfma > gpurun_out/s4_dfma.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/s4_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/s4_tests.log
timeout 300 python tools/fixed_cost_probe.py > gpurun_out/s4_probe.log 2>&1
timeout 300 python tools/timeline_f32.py C1 > gpurun_out/s4_tl_c1.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/s4_bench.log 2>&1
cat gpurun_out/s4_dfma.log; tail -5 gpurun_out/s4_tests.log; cat gpurun_out/s4_probe.log; tail -8 gpurun_out/s4_tl_c1.log; tail -1 gpurun_out/s4_bench.log | cut -c1-300
