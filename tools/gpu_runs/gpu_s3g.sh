#!/bin/bash
mkdir -p gpurun_out
CMD="python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --lanes 1 --reserve-sms 0"
timeout 1500 ncu --nvtx --nvtx-include "gift.query_batch/" --set full --import-source on --clock-control none -k regex:owner_reduce -s 2 -c 1 -o gpurun_out/s3g_own $CMD > gpurun_out/s3g_ncu.log 2>&1; echo ncu=$?
