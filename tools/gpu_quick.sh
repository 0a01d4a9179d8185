#!/bin/bash
# quick GPU check: gpu tests + bench summary (run under gpurun)
timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 400 python bench.py --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
r=d['roofline']
print('step_ms', d['ms_per_step'], 'tok/s', d['value'], 'partial_ms', r['kernel_ms'], 'GB/s', r['achieved'], 'frac', r['frac'], 'e2e', d['e2e']['value'], 'clocks', d['clocks'])"
