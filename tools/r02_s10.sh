#!/bin/bash
# state mode + decode PDL + graph replay: graph tests, full GPU suite, probe (eager vs graph), timelines
mkdir -p gpurun_out
tag=s10
timeout 600 python -m pytest tests/test_gpu_graph.py -x -q -m gpu > gpurun_out/${tag}_graph_tests.log 2>&1; echo "rc $?" >> gpurun_out/${tag}_graph_tests.log
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/${tag}_tests.log
timeout 300 python tools/fixed_cost_probe.py > gpurun_out/${tag}_probe.log 2>&1
timeout 600 ncu --nvtx --nvtx-include "timed_graph/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_launch.csv python tools/fixed_cost_probe.py C1 > gpurun_out/${tag}_launch_run.log 2>&1
python tools/launch_summary.py gpurun_out/${tag}_launch.csv > gpurun_out/${tag}_launch_summary.txt 2>&1
for c in EMPTY C1; do timeout 300 python tools/timeline_f32.py $c > gpurun_out/${tag}_tl_$c.log 2>&1; done
tail -15 gpurun_out/${tag}_graph_tests.log; tail -3 gpurun_out/${tag}_tests.log; cat gpurun_out/${tag}_probe.log gpurun_out/${tag}_launch_summary.txt
tail -6 gpurun_out/${tag}_tl_EMPTY.log; tail -8 gpurun_out/${tag}_tl_C1.log
