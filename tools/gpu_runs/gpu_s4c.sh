#!/bin/bash
# full GPU suite (config-scale HBM release fix) + C4 timeline
mkdir -p gpurun_out
export GIFT_PARITY_OUT=gpurun_out/s4c_parity.jsonl
timeout 2400 python -m pytest tests -m gpu -q --durations=40 > gpurun_out/s4c_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/s4c_tests.log
grep -E "^FAILED|^ERROR" gpurun_out/s4c_tests.log | head
bash tools/gpu_runs/gpu_s4b.sh
