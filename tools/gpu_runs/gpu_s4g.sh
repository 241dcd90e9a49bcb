#!/bin/bash
# f64 query_fif path: parity tests + the reference's own suite against the shim
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "f64 or query_fif or zero_views" > gpurun_out/s4g_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/s4g_tests.log
GIFT_REFSUITE_OUT=gpurun_out/s4g_reference_suite.txt timeout 1500 python -m pytest tests/test_gpu_reference_suite.py -q -x > gpurun_out/s4g_refsuite.log 2>&1; echo refsuite=$?
tail -3 gpurun_out/s4g_refsuite.log
grep -E "FAILED|passed|failed" gpurun_out/s4g_reference_suite.txt | tail -8
