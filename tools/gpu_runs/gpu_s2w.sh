#!/bin/bash
# owner reduce variants (loads per round x CTAs per SM) on config 4
mkdir -p gpurun_out
cp paper_1604_01879_b200/libgift.so /tmp/libgift_prod.so
for v in 16_4 16_3 8_3 4_4; do
cp tools/libgift_own_$v.so paper_1604_01879_b200/libgift.so
CMD="python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --lanes 1 --reserve-sms 0"
timeout 1500 ncu --nvtx --nvtx-include "gift.query_batch/" -k regex:owner_reduce --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2w_own_$v.csv $CMD > /dev/null 2>&1; echo $v=$?
python tools/launch_table.py gpurun_out/s2w_own_$v.csv | sed -n 2p
done
cp /tmp/libgift_prod.so paper_1604_01879_b200/libgift.so
