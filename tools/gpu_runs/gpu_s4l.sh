#!/bin/bash
# ncu --set full of C5's S-IF kernels (one batch each, lanes 1)
mkdir -p gpurun_out
CMD5="python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --lanes 1"
timeout 900 $CMD5 > gpurun_out/s4l_plain.json 2>&1; echo plain=$?
for k in sif_split sif_bucket_reduce sif_bucket_rank; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/s4l_$k $CMD5 > gpurun_out/s4l_ncu_$k.log 2>&1; echo ncu_$k=$?
ncu -i gpurun_out/s4l_$k.ncu-rep --page raw --csv > gpurun_out/s4l_${k}_metrics.csv 2>/dev/null
ncu -i gpurun_out/s4l_$k.ncu-rep --page details --csv > gpurun_out/s4l_${k}_details.csv 2>/dev/null
done
