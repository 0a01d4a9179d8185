#!/bin/bash
mkdir -p gpurun_out
tag=s15
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/${tag}_tests.log
timeout 300 python tools/fixed_cost_probe.py > gpurun_out/${tag}_probe.log 2>&1
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
tail -3 gpurun_out/${tag}_tests.log; cat gpurun_out/${tag}_probe.log
python - <<'PY'
import json
d=json.loads(open("gpurun_out/s15_bench.json").read().strip().splitlines()[-1])
print("C3", d["value"], d["ms_per_step"], d["roofline"]["frac"], d["roofline"]["kernel_ms"], "e2e", d["e2e"]["value"], "C2", d["c2"]["value"], d["c2"]["roofline_frac"])
PY
