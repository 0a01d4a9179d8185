#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_acceptance.py -q -m gpu > gpurun_out/s3_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/s3_tests.log
grep -E "passed|failed|Error|assert" gpurun_out/s3_tests.log | tail -30
