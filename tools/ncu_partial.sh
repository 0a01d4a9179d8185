#!/bin/bash
# ncu --set full capture of one decode_partial launch from the C2 bench (run under gpurun).
# usage: tools/ncu_partial.sh <tag>
tag=${1:-prof}
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_partial -s 520 -c 1 \
  -o gpurun_out/${tag} python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/${tag}_log.txt 2>&1
tail -2 gpurun_out/${tag}_log.txt | cut -c1-300
