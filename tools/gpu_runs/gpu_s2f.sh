#!/bin/bash
mkdir -p gpurun_out
cp paper_1604_01879_b200/libgift.so /tmp/libgift_prod.so
timeout 600 python tools/scan_trace.py c4s > gpurun_out/s2f_trace_c4s.log 2>&1; echo trace=$?
timeout 600 python tools/scan_trace.py c4s 8 > gpurun_out/s2f_trace_c4s_d8.log 2>&1; echo trace=$?
timeout 600 python tools/scan_trace.py c4s 0 32 > gpurun_out/s2f_trace_c4s_nop1.log 2>&1; echo trace=$?
timeout 600 python tools/scan_trace.py c4s 0 1 > gpurun_out/s2f_trace_c4s_notail.log 2>&1; echo trace=$?
cp /tmp/libgift_prod.so paper_1604_01879_b200/libgift.so
