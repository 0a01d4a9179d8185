#!/bin/bash
# bench each library variant (run under gpurun): tools/gpu_variants.sh "" p1 p3
L=paper_2507_03153_b200/_lib
for v in "$@"; do
  lib=$L/libhgca_b200${v:+_$v}.so
  echo "=== bench [$v]"; HGCA_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --steps 200 --e2e-steps 20 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('step_ms', d['ms_per_step'], 'kernel_ms', r['kernel_ms'], 'GB/s', r['achieved'], 'frac', r['frac'])"
done
