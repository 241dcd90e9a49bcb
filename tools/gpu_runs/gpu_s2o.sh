#!/bin/bash
mkdir -p gpurun_out
cp paper_1604_01879_b200/libgift.so /tmp/libgift_prod.so
timeout 600 python tools/scan_trace.py c4s 0 0 1 > gpurun_out/s2o_trace_dense.log 2>&1; echo trace=$?
timeout 600 python tools/scan_trace.py c4s 8 0 1 > gpurun_out/s2o_trace_dense_d8.log 2>&1; echo trace=$?
cp /tmp/libgift_prod.so paper_1604_01879_b200/libgift.so
