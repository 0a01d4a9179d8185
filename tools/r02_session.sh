#!/bin/bash
# Round-2 GPU session: gpu tests, smoke, bench (N=1), reference arm, launch list of the timed steps.
tag=${1:-r02x}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${tag}_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.txt
tail -4 gpurun_out/${tag}_pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/${tag}_smoke.txt 2>&1; tail -2 gpurun_out/${tag}_smoke.txt
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; tail -c 4000 gpurun_out/${tag}_bench.json; tail -5 gpurun_out/${tag}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err; tail -c 1500 gpurun_out/${tag}_bench_ref.json
bash tools/launch_list.sh ${tag}_launches 20 > /dev/null 2>&1; tail -30 gpurun_out/${tag}_launches_summary.txt
