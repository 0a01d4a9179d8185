#!/bin/bash
# per-launch device times of the bench's steady-state steps (run under gpurun)
tag=${1:-launches}
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -s 3700 -c ${2:-200} --csv \
  --log-file gpurun_out/${tag}.csv python bench.py --steps 60 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${tag}.csv
