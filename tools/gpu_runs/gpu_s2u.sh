#!/bin/bash
# C4: lanes / reserved-SM sweep, launch list of the query batches, ncu --set full of the dense scan
mkdir -p gpurun_out
for cfg in "1 0" "2 0" "2 8" "2 20" "3 20"; do set -- $cfg
timeout 1200 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline --lanes $1 --reserve-sms $2 > gpurun_out/s2u_c4_l$1_r$2.json 2>/dev/null
tail -1 gpurun_out/s2u_c4_l$1_r$2.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c4 lanes $1 reserve $2', round(d['value']), round(d['e2e']['value']), round(r['scan_ms_avg'],2), round(d['ms_per_step'],2))"
done
CMD="python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --lanes 1 --reserve-sms 0"
timeout 1500 ncu --nvtx --nvtx-include "gift.query_batch/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2u_launches_c4.csv $CMD > gpurun_out/s2u_ncu1.log 2>&1; echo launches=$?
timeout 1500 ncu --nvtx --nvtx-include "gift.query_batch/" --set full --import-source on --clock-control none -k regex:fif_scan_dense -s 1 -c 1 -o gpurun_out/s2u_dense_c4 $CMD > gpurun_out/s2u_ncu2.log 2>&1; echo full=$?
tail -2 gpurun_out/s2u_ncu2.log
