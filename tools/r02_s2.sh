#!/bin/bash
# round-2 GPU session 2: new API / acceptance / C1 tests + fp32 timeline
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_acceptance.py tests/test_gpu_c1.py -x -q -m gpu > gpurun_out/s2_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/s2_tests.log
timeout 300 python tools/timeline_f32.py C1 > gpurun_out/s2_tl_c1.log 2>&1
timeout 300 python tools/timeline_f32.py EMPTY > gpurun_out/s2_tl_empty.log 2>&1
tail -30 gpurun_out/s2_tests.log; cat gpurun_out/s2_tl_c1.log gpurun_out/s2_tl_empty.log | tail -30
