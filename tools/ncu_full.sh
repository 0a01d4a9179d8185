#!/bin/bash
# one ncu --set full capture per kernel of a steady-state bench decode step (run under gpurun)
tag=${1:-r01}
skip=${2:-2}   # launches of the kernel to skip inside the timed NVTX range
mkdir -p gpurun_out
for k in ${KERNELS:-decode_bf16 decode_merge}; do
  timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" -k regex:${k} -s ${skip:-2} -c 1 \
    -o gpurun_out/${tag}_${k} python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 \
    > gpurun_out/${tag}_${k}_log.txt 2>&1
  python tools/ncu_summary.py gpurun_out/${tag}_${k}.ncu-rep 25 > gpurun_out/${tag}_${k}_summary.txt 2>&1
  head -32 gpurun_out/${tag}_${k}_summary.txt
done
