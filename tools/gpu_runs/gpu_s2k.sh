#!/bin/bash
mkdir -p gpurun_out
cp paper_1604_01879_b200/libgift.so /tmp/libgift_prod.so
for b in 0 16; do
timeout 600 python tools/scan_trace.py c4s 0 $b > gpurun_out/s2k_trace_c4s_$b.log 2>&1; echo trace=$?
grep "scan\|median\|tail parts" gpurun_out/s2k_trace_c4s_$b.log | head -4
done
cp /tmp/libgift_prod.so paper_1604_01879_b200/libgift.so
