#!/bin/bash
# per-role scan timeline (experiment build) on c4s and c4
mkdir -p gpurun_out
timeout 600 python tools/scan_trace.py c4s > gpurun_out/s2b_trace_c4s.log 2>&1; echo c4s=$?
timeout 600 python tools/scan_trace.py c4s 8 > gpurun_out/s2b_trace_c4s_d8.log 2>&1; echo c4s8=$?
timeout 900 python tools/scan_trace.py c4 > gpurun_out/s2b_trace_c4.log 2>&1; echo c4=$?
