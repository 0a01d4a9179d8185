#!/bin/bash
# per-launch device times of the bench's timed steps only (NVTX range "timed"); run under gpurun
tag=${1:-launches}
timeout 600 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}.csv python bench.py --steps ${2:-20} --warmup 3 --no-cpu-baseline --e2e-steps 2 \
  > gpurun_out/${tag}_bench.log 2>&1
python tools/launch_summary.py gpurun_out/${tag}.csv | tee gpurun_out/${tag}_summary.txt
