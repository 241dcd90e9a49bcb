#!/bin/bash
mkdir -p gpurun_out
CMD="python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --sif hash"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sif_hash -s 3 -c 1 -o gpurun_out/s3d_hash $CMD > gpurun_out/s3d_ncu.log 2>&1; echo ncu=$?
