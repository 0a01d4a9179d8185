#!/bin/bash
# GPU tests + the other BASELINE configs (eager and graph mode)
mkdir -p gpurun_out
tag=${1:-cfg}
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${tag}_tests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_tests.txt
tail -3 gpurun_out/${tag}_tests.txt
for c in ${CFGS:-C1 C5S C3 C4}; do timeout 900 python tools/bench_configs.py $c >> gpurun_out/${tag}_configs.jsonl 2> gpurun_out/${tag}_configs_$c.err; done
cat gpurun_out/${tag}_configs.jsonl
