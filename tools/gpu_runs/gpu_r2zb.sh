#!/bin/bash
# ncu --set full of the bucketed S-IF kernels (one launch each) on config 5
mkdir -p gpurun_out
CMD="python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --sif bucket"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"sif_split" -c 1 -o gpurun_out/r2zf_sif $CMD > gpurun_out/r2zf_ncu.log 2>&1; echo ncu=$?
tail -3 gpurun_out/r2zf_ncu.log
