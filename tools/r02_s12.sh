#!/bin/bash
mkdir -p gpurun_out
tag=s12
timeout 600 python -m pytest tests/test_gpu_graph.py -x -q -m gpu > gpurun_out/${tag}_graph_tests.log 2>&1; echo "rc $?" >> gpurun_out/${tag}_graph_tests.log
timeout 300 python tools/fixed_cost_probe.py > gpurun_out/${tag}_probe.log 2>&1
tail -15 gpurun_out/${tag}_graph_tests.log; cat gpurun_out/${tag}_probe.log
