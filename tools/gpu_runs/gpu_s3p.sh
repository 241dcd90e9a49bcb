#!/bin/bash
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_small.py > gpurun_out/s3p_$tool.log 2>&1; echo $tool=$?
grep -E "ERROR SUMMARY|workload done|Error|error" gpurun_out/s3p_$tool.log | head -5
done
