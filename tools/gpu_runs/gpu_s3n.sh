#!/bin/bash
# dense-cell threshold: 128 / 192 (default) / 256 probes
mkdir -p gpurun_out
cp paper_1604_01879_b200/libgift.so /tmp/libgift_prod.so
for v in 192 128 256; do
if [ $v != 192 ]; then cp tools/libgift_dense_$v.so paper_1604_01879_b200/libgift.so; else cp /tmp/libgift_prod.so paper_1604_01879_b200/libgift.so; fi
CMD="python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --lanes 1 --reserve-sms 0"
timeout 1500 ncu --nvtx --nvtx-include "gift.query_batch/" -k regex:fif_scan --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3n_$v.csv $CMD > /dev/null 2>&1; echo d$v=$?
python tools/launch_table.py gpurun_out/s3n_$v.csv | sed -n 2,4p
done
cp /tmp/libgift_prod.so paper_1604_01879_b200/libgift.so
