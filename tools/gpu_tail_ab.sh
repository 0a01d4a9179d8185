#!/bin/bash
# tail-share A/B (HGCA_TAIL_DIV build variants) on graph-mode steps: C4 layer, C3, C2-shape, C5 small
for v in ${VARIANTS:-base td4 td3 td2}; do
  lib=paper_2507_03153_b200/_lib/libhgca_b200.so; [ $v != base ] && lib=paper_2507_03153_b200/_lib/libhgca_b200_$v.so
  echo "== $v"; HGCA_LIB=$lib python tools/fixed_cost_probe.py C4L C5S 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['cfg'], 'graph us/step', d['graph_device_us_per_step'], 'eager', d['device_us_per_step'])"
  HGCA_LIB=$lib python tools/bench_configs.py C3 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('C3 graph us/step', round(d['graph_ms_per_step']*1e3,2), 'pair', round(d['layer_step_kernel_ms']*1e3,2))"
done
