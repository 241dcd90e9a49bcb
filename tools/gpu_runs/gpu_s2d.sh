#!/bin/bash
# tail experiments on c4s (experiment build): full, no stores, no pass 1, no tail
mkdir -p gpurun_out
cp paper_1604_01879_b200/libgift.so /tmp/libgift_prod.so
for b in 0 16 32 48 1; do
timeout 600 python tools/scan_trace.py c4s 0 $b > gpurun_out/s2d_trace_$b.log 2>&1; echo trace$b=$?
grep "scan\|median" gpurun_out/s2d_trace_$b.log | head -4
done
cp /tmp/libgift_prod.so paper_1604_01879_b200/libgift.so
