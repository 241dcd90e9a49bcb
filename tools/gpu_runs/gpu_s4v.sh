#!/bin/bash
# C2 full-scale cosine + f64-path parity (new test)
mkdir -p gpurun_out
export GIFT_PARITY_OUT=gpurun_out/s4v_parity.jsonl
timeout 1200 python -m pytest tests/test_gpu_config_scale.py -q -k "TestC2" > gpurun_out/s4v_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/s4v_tests.log
cat gpurun_out/s4v_parity.jsonl
