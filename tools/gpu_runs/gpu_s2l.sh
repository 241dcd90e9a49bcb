#!/bin/bash
# ncu --set full of the dense scan on c4s (one launch), for per-instruction stall sampling
mkdir -p gpurun_out
CMD="python bench.py --config c4s --steps 1 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/s2l_plain.json 2> gpurun_out/s2l_plain.err; echo plain=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fif_scan_dense -s 2 -c 1 -o gpurun_out/s2l_dense $CMD > gpurun_out/s2l_ncu.log 2>&1; echo ncu=$?
tail -3 gpurun_out/s2l_ncu.log
