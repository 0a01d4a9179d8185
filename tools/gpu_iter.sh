#!/bin/bash
# quick GPU iteration: build (incl. timeline variant), gpu tests, timeline, bench (run under gpurun)
python paper_2507_03153_b200/_build.py --timeline > /dev/null 2>&1
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
timeout 300 python tools/timeline.py 2>&1 | tail -12
timeout 400 python bench.py --no-cpu-baseline --steps 200 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
r=d['roofline']
print('step_ms', d['ms_per_step'], 'tok/s', d['value'], 'kernel_ms', r['kernel_ms'], 'GB/s', r['achieved'], 'frac', r['frac'], 'e2e', d['e2e']['value'], 'clocks', d['clocks'])"
