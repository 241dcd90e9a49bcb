#!/bin/bash
# C5 S-IF split grid: 1 / 2 / 4 CTAs per SM
mkdir -p gpurun_out
cp paper_1604_01879_b200/libgift.so /tmp/libgift_prod.so
for v in 1 2 4; do
if [ $v != 1 ]; then cp tools/libgift_sb_$v.so paper_1604_01879_b200/libgift.so; else cp /tmp/libgift_prod.so paper_1604_01879_b200/libgift.so; fi
timeout 900 python bench.py --config c5 --steps 12 --warmup 3 --no-cpu-baseline > gpurun_out/s3o_$v.json 2>/dev/null; echo sb$v=$?
tail -1 gpurun_out/s3o_$v.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('grid x$v', round(d['value']), round(d['e2e']['value']), d['roofline']['sif_ms_avg'])"
done
cp /tmp/libgift_prod.so paper_1604_01879_b200/libgift.so
