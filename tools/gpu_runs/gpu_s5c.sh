#!/bin/bash
# session 5: the reference's own suite against the shim on the restaged copy
mkdir -p gpurun_out
export GIFT_REFSUITE_OUT=gpurun_out/s5c_reference_suite.txt
timeout 1200 python -m pytest tests/test_gpu_reference_suite.py -m gpu -q > gpurun_out/s5c_tests.log 2>&1; echo tests=$?
tail -1 gpurun_out/s5c_tests.log
tail -1 gpurun_out/s5c_reference_suite.txt
