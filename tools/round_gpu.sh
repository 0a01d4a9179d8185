#!/bin/bash
# One GPU session: gpu tests, smoke, bench (N=1, with cpu baseline), reference arm,
# launch list and one ncu --set full capture of the decode kernel.  (run under gpurun)
tag=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/${tag}_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.txt
tail -3 gpurun_out/${tag}_pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/${tag}_smoke.txt 2>&1; tail -2 gpurun_out/${tag}_smoke.txt
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; tail -c 3000 gpurun_out/${tag}_bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err; tail -c 1500 gpurun_out/${tag}_bench_ref.json
timeout 500 ncu --metrics gpu__time_duration.sum --clock-control none -s 3700 -c 200 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 60 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${tag}_launches.csv
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_partial -s 520 -c 1 \
  -o gpurun_out/${tag}_decode python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/${tag}_ncu_log.txt 2>&1
ls -la gpurun_out/
