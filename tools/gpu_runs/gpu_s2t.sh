#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_streamed.py -q > gpurun_out/s2t.log 2>&1; echo tests=$?
grep -E "passed|failed|Error|Mismatch" gpurun_out/s2t.log | head -20
