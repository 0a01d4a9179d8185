#!/bin/bash
# fp32 decode warp-specialized: tests touching the fp32 path, probe, timelines
mkdir -p gpurun_out
tag=s9
./tools/bin/probe_dfma > gpurun_out/${tag}_dfma.log 2>&1
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_c1.py tests/test_gpu_kernels.py -x -q -m gpu > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/${tag}_tests.log
timeout 300 python tools/fixed_cost_probe.py > gpurun_out/${tag}_probe.log 2>&1
timeout 600 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_launch.csv python tools/fixed_cost_probe.py EMPTY C1 > gpurun_out/${tag}_launch_run.log 2>&1
python tools/launch_summary.py gpurun_out/${tag}_launch.csv > gpurun_out/${tag}_launch_summary.txt 2>&1
for c in EMPTY C1; do timeout 300 python tools/timeline_f32.py $c > gpurun_out/${tag}_tl_$c.log 2>&1; done
cat gpurun_out/${tag}_dfma.log; tail -3 gpurun_out/${tag}_tests.log; cat gpurun_out/${tag}_probe.log gpurun_out/${tag}_launch_summary.txt
tail -6 gpurun_out/${tag}_tl_EMPTY.log; tail -8 gpurun_out/${tag}_tl_C1.log
