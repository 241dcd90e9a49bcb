#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/graph_probe.py c1 > gpurun_out/s3l_c1.log 2>&1; echo c1=$?
tail -4 gpurun_out/s3l_c1.log
timeout 600 python tools/graph_probe.py c2 > gpurun_out/s3l_c2.log 2>&1; echo c2=$?
tail -4 gpurun_out/s3l_c2.log
