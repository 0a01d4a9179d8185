#!/bin/bash
# round-2 (session 2) GPU evidence: tests, smoke, bench + reference arm, launch list,
# ncu --set full of the decode and merge kernels, fixed-cost probe. (run under gpurun)
tag=r02a
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
lscpu | head -20 > gpurun_out/${tag}_lscpu.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/${tag}_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/${tag}_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err
timeout 300 python tools/fixed_cost_probe.py > gpurun_out/${tag}_probe.log 2>&1
timeout 600 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-c2 --e2e-steps 2 > gpurun_out/${tag}_launches_bench.log 2>&1
python tools/launch_summary.py gpurun_out/${tag}_launches.csv > gpurun_out/${tag}_launches_summary.txt 2>&1
KERNELS="decode_bf16 decode_merge" bash tools/ncu_full.sh ${tag} 2 > /dev/null 2>&1
tail -3 gpurun_out/${tag}_pytest_gpu.txt; tail -2 gpurun_out/${tag}_smoke.txt
tail -c 2500 gpurun_out/${tag}_bench.json; tail -c 800 gpurun_out/${tag}_bench_ref.json
cat gpurun_out/${tag}_probe.log gpurun_out/${tag}_launches_summary.txt
head -30 gpurun_out/${tag}_decode_bf16_summary.txt
