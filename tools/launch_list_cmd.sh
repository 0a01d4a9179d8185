#!/bin/bash
# per-launch device times inside NVTX range "timed" of any command; run under gpurun
#   tools/launch_list_cmd.sh TAG python tools/bench_configs.py C4L
tag=$1; shift
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}.csv "$@" > gpurun_out/${tag}_run.log 2>&1
python tools/launch_summary.py gpurun_out/${tag}.csv | tee gpurun_out/${tag}_summary.txt
