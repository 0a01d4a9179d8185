#!/bin/bash
# round-2 final evidence: GPU tests, smoke, default bench line, reference arm, launch list,
# ncu --set full of the C3 step kernels, memcheck of the decode and graph paths
mkdir -p gpurun_out
tag=${1:-fin}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${tag}_tests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_tests.txt
tail -3 gpurun_out/${tag}_tests.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/${tag}_smoke.txt 2>&1; tail -1 gpurun_out/${tag}_smoke.txt
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; tail -c 600 gpurun_out/${tag}_bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err; tail -c 400 gpurun_out/${tag}_bench_ref.json
bash tools/launch_list.sh ${tag}_launches 20 > /dev/null 2>&1; head -9 gpurun_out/${tag}_launches_summary.txt
KERNELS="decode_bf16 decode_merge" bash tools/ncu_full.sh ${tag} 2 > /dev/null 2>&1
for k in decode_bf16 decode_merge; do head -6 gpurun_out/${tag}_${k}_summary.txt; done
for m in bf16-decode f32 graph; do
  timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_run.py $m > gpurun_out/${tag}_memcheck_$m.txt 2>&1
  echo "memcheck $m: $(grep -h 'ERROR SUMMARY' gpurun_out/${tag}_memcheck_$m.txt | tail -1)"
done
