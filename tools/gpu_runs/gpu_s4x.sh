#!/bin/bash
# thread-local pinned buffers: query_many tests + C1 bench (graph lanes, e2e)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_streamed.py -q -k "query_many or streamed" > gpurun_out/s4x_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/s4x_tests.log
timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/s4x_c1.json 2>/dev/null; grep "^{" gpurun_out/s4x_c1.json | tail -1 | cut -c1-200
