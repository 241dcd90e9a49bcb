#!/bin/bash
# ncu evidence on the current code: C2 query-batch scan + quantizer (--set full),
# C2 query-batch launch list with DRAM bytes, C5 S-IF launch list with DRAM bytes
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/s4f_plain_c2.json 2>&1; echo plain=$?
NV="--nvtx --nvtx-include gift.query_batch/"
timeout 900 ncu --set full --clock-control none --import-source on $NV -k regex:fif_scan_tc -s 3 -c 1 -o gpurun_out/s4f_scan_c2 $CMD > gpurun_out/s4f_ncu1.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on $NV -k regex:quant_approx_tc -s 3 -c 1 -o gpurun_out/s4f_quant_c2 $CMD > gpurun_out/s4f_ncu2.log 2>&1; echo ncu2=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none $NV --csv --log-file gpurun_out/s4f_launches_c2.csv $CMD > gpurun_out/s4f_ncu3.log 2>&1; echo ncu3=$?
for r in s4f_scan_c2 s4f_quant_c2; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_metrics.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null
done
ncu -i gpurun_out/s4f_scan_c2.ncu-rep --page source --csv > gpurun_out/s4f_scan_c2_source.csv 2>/dev/null
CMD5="python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --lanes 1"
timeout 900 $CMD5 > gpurun_out/s4f_plain_c5.json 2>&1; echo plain5=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:sif_ --csv --log-file gpurun_out/s4f_launches_c5.csv $CMD5 > gpurun_out/s4f_ncu5.log 2>&1; echo ncu5=$?
ls -la gpurun_out/ | grep s4f
