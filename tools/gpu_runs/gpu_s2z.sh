#!/bin/bash
mkdir -p gpurun_out
CMD="python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s2z_launches_c5.csv $CMD > gpurun_out/s2z_ncu.log 2>&1; echo launches=$?
