#!/bin/bash
# round-2 evidence session: GPU tests, compute-sanitizer on every kernel family (incl. graph mode),
# ncu --set full of the C3 step kernels and of the C1 fp32 kernel, launch list of the bench's timed steps
mkdir -p gpurun_out
tag=${1:-ev}
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${tag}_tests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_tests.txt
tail -3 gpurun_out/${tag}_tests.txt
for m in bf16-decode bf16-append bf16-append-tc5 bf16-append-tc5x2 f32 graph; do
  timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_run.py $m > gpurun_out/${tag}_memcheck_$m.txt 2>&1
  echo "memcheck $m: $(grep -h 'ERROR SUMMARY' gpurun_out/${tag}_memcheck_$m.txt | tail -1)"
done
for m in f32 graph; do
  timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_run.py $m > gpurun_out/${tag}_racecheck_$m.txt 2>&1
  echo "racecheck $m: $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' gpurun_out/${tag}_racecheck_$m.txt | tail -2 | tr '\n' ' ')"
done
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_run.py f32 > gpurun_out/${tag}_synccheck_f32.txt 2>&1
echo "synccheck f32: $(grep -h 'ERROR SUMMARY' gpurun_out/${tag}_synccheck_f32.txt | tail -1)"
bash tools/launch_list.sh ${tag}_launches 20 > /dev/null 2>&1; head -12 gpurun_out/${tag}_launches_summary.txt
KERNELS="decode_bf16 decode_merge" bash tools/ncu_full.sh ${tag} 2 > /dev/null 2>&1
for k in decode_bf16 decode_merge; do head -22 gpurun_out/${tag}_${k}_summary.txt; done
timeout 600 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" -k regex:decode_f32 -s 20 -c 1 \
    -o gpurun_out/${tag}_c1_decode_f32 python tools/fixed_cost_probe.py C1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${tag}_c1_decode_f32.ncu-rep 25 > gpurun_out/${tag}_c1_decode_f32_summary.txt 2>&1
head -22 gpurun_out/${tag}_c1_decode_f32_summary.txt
