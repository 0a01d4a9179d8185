#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/s5_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/s5_tests.log
timeout 300 python tools/fixed_cost_probe.py > gpurun_out/s5_probe.log 2>&1
timeout 300 python tools/timeline_f32.py C1 > gpurun_out/s5_tl_c1.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/s5_bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/s5_bench_ref.log 2>&1
tail -5 gpurun_out/s5_tests.log; cat gpurun_out/s5_probe.log; tail -7 gpurun_out/s5_tl_c1.log; tail -1 gpurun_out/s5_bench.log; tail -1 gpurun_out/s5_bench_ref.log
