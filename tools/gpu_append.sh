#!/bin/bash
# append / re-evaluation: GPU tests touching it + per-kernel launch times of tools/append_probe.py (C2 scale)
mkdir -p gpurun_out
tag=${1:-app}
timeout 900 python -m pytest tests -x -q -m gpu -k "append or reeval or soak or acceptance" > gpurun_out/${tag}_tests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_tests.txt
tail -3 gpurun_out/${tag}_tests.txt
timeout 600 python tools/append_probe.py > gpurun_out/${tag}_probe.txt 2>&1; cat gpurun_out/${tag}_probe.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:append --csv --log-file gpurun_out/${tag}_launch.csv python tools/append_probe.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${tag}_launch.csv | head -20
