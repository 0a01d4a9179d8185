#!/bin/bash
# C1 (fp32, reference-exact kernels) step anatomy: graph-mode gap probe + ncu --set full of both step kernels
mkdir -p gpurun_out
tag=${1:-c1}
HGCA_LIB=paper_2507_03153_b200/_lib/libhgca_b200_tl.so timeout 300 python tools/gap_probe.py ${CFGS:-C1 C1B C5S} > gpurun_out/${tag}_gaps.txt 2>&1
for k in decode_f32 decode_merge; do
  timeout 600 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" -k regex:${k} -s 20 -c 1 \
    -o gpurun_out/${tag}_${k} python tools/fixed_cost_probe.py C1 > gpurun_out/${tag}_${k}_log.txt 2>&1
  python tools/ncu_summary.py gpurun_out/${tag}_${k}.ncu-rep 30 > gpurun_out/${tag}_${k}_summary.txt 2>&1
done
cat gpurun_out/${tag}_gaps.txt; head -45 gpurun_out/${tag}_decode_f32_summary.txt; head -45 gpurun_out/${tag}_decode_merge_summary.txt
