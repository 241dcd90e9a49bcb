#!/bin/bash
mkdir -p gpurun_out
cp paper_1604_01879_b200/libgift.so /tmp/libgift_prod.so
timeout 600 python tools/scan_trace.py c4s > gpurun_out/s2h_trace_c4s.log 2>&1; echo trace=$?
head -4 gpurun_out/s2h_trace_c4s.log
cp /tmp/libgift_prod.so paper_1604_01879_b200/libgift.so
