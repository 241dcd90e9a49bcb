#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_sharded.py -q -x > gpurun_out/s3a.log 2>&1; echo tests=$?
grep -E "passed|failed|Error" gpurun_out/s3a.log | head -10
