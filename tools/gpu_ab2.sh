#!/bin/bash
# GPU tests + small-step anatomy (gap probe, fixed-cost probe) for the current build and the S=1 fp32 variant
mkdir -p gpurun_out
tag=${1:-ab2}
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${tag}_tests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_tests.txt
tail -4 gpurun_out/${tag}_tests.txt
HGCA_LIB=paper_2507_03153_b200/_lib/libhgca_b200_tl.so timeout 300 python tools/gap_probe.py EMPTY EMPTYB C1 C1B C5S > gpurun_out/${tag}_gaps.txt 2>&1
timeout 300 python tools/fixed_cost_probe.py > gpurun_out/${tag}_probe.txt 2>&1
HGCA_LIB=paper_2507_03153_b200/_lib/libhgca_b200_s1.so timeout 300 python tools/fixed_cost_probe.py C1 EMPTY > gpurun_out/${tag}_probe_s1.txt 2>&1
cat gpurun_out/${tag}_gaps.txt gpurun_out/${tag}_probe.txt gpurun_out/${tag}_probe_s1.txt
