#!/bin/bash
# shim warm-up at import: the reference suite twice; f64 chunking test
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "f64" > gpurun_out/s4t_f64.log 2>&1; echo f64=$?; tail -1 gpurun_out/s4t_f64.log
for i in 1 2; do
GIFT_REFSUITE_OUT=gpurun_out/s4t_reference_suite_$i.txt timeout 1500 python -m pytest tests/test_gpu_reference_suite.py -q > gpurun_out/s4t_refsuite_$i.log 2>&1; echo refsuite=$?
grep -E "criterion 1|passed|failed" gpurun_out/s4t_reference_suite_$i.txt | tail -3
done
