#!/bin/bash
# C5 with S-IF batches in flight
mkdir -p gpurun_out
for L in 1 2 3 4; do
timeout 900 python bench.py --config c5 --steps 12 --warmup 3 --no-cpu-baseline --lanes $L > gpurun_out/s3j_c5_l$L.json 2> gpurun_out/s3j_c5_l$L.err; echo c5_$L=$?
tail -1 gpurun_out/s3j_c5_l$L.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lanes $L', round(d['value']), round(d['e2e']['value']), d['ms_per_step'])"
done
tail -3 gpurun_out/s3j_c5_l2.err
