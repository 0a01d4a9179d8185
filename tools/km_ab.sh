#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "append or reeval or soak or acceptance" > gpurun_out/km_tests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/km_tests.txt
tail -3 gpurun_out/km_tests.txt
for v in ${KM_VARIANTS:-new old nt1}; do
  case $v in new) E="";; old) E="HGCA_APPEND_MEAN_OLD=1";; nt1) E="HGCA_APPEND_MEAN_NT=1";; nosplit) E="HGCA_APPEND_SPLIT_KEYS=0";; esac
  env $E HGCA_APPEND_NQ=16,64,16,64 timeout 600 python tools/append_probe.py > gpurun_out/km_probe_$v.txt 2>&1; echo "== $v"; cat gpurun_out/km_probe_$v.txt | tail -4
  env $E HGCA_APPEND_NQ=16,64 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:append --csv --log-file gpurun_out/km_launch_$v.csv python tools/append_probe.py > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/km_launch_$v.csv | head -8
done
