#!/bin/bash
# C5 bucket reduce: bucket width (2^rb shapes) x reducing CTAs per SM; parity per variant
mkdir -p gpurun_out
cp paper_1604_01879_b200/libgift.so /tmp/libgift_prod.so
for v in D F G H I; do
if [ $v != P ]; then cp tools/libgift_sb$v.so paper_1604_01879_b200/libgift.so; else cp /tmp/libgift_prod.so paper_1604_01879_b200/libgift.so; fi
timeout 600 python -m pytest tests/test_gpu_config_scale.py -q -x -k c5 > gpurun_out/s4k_t_$v.log 2>&1; echo "$v tests=$? $(tail -1 gpurun_out/s4k_t_$v.log)"
for L in 3 1; do
timeout 900 python bench.py --config c5 --steps 12 --warmup 3 --no-cpu-baseline --lanes $L > gpurun_out/s4k_c5_${v}_$L.json 2>/dev/null
grep "^{" gpurun_out/s4k_c5_${v}_$L.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('variant $v lanes $L', round(d['value']), round(d['e2e']['value']), d['roofline']['sif_ms_avg'])"
done
done
cp /tmp/libgift_prod.so paper_1604_01879_b200/libgift.so
