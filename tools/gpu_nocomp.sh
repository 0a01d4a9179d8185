#!/bin/bash
L=paper_2507_03153_b200/_lib
for v in nocomp nocomps1 nocomps3 nocomps4; do
  echo "=== bench [$v]"; HGCA_LIB=$L/libhgca_b200_$v.so timeout 300 python bench.py --no-cpu-baseline --steps 100 --e2e-steps 5 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('step_ms', d['ms_per_step'], 'kernel_ms', r['kernel_ms'], 'GB/s', r['achieved'], 'frac', r['frac'])"
done
echo "=== timeline nocomp"; HGCA_LIB=$L/libhgca_b200_tlnocomp.so timeout 300 python tools/timeline.py 2>&1 | tail -7
