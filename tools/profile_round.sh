#!/bin/bash
# ncu evidence for one round (run under gpurun; single GPU, never multi-rank):
#   launch list of a short bench run (per-launch device times, cold/serialised)
#   + one --set full capture of the decode kernel and of the merge kernel.
tag=${1:-r01}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 \
  > gpurun_out/${tag}_launches_bench.log 2>&1
python tools/launch_summary.py gpurun_out/${tag}_launches.csv 60 > gpurun_out/${tag}_launches_summary.txt
cat gpurun_out/${tag}_launches_summary.txt
for k in decode_bf16 decode_merge; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:${k} -s 600 -c 1 \
    -o gpurun_out/${tag}_${k} python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 \
    > gpurun_out/${tag}_${k}_log.txt 2>&1
  python tools/ncu_summary.py gpurun_out/${tag}_${k}.ncu-rep 25 > gpurun_out/${tag}_${k}_summary.txt 2>&1
  head -30 gpurun_out/${tag}_${k}_summary.txt
done
