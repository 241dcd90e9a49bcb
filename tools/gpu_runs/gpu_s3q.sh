#!/bin/bash
# concurrent dense / other-cells scans: tests, C4 lanes x side SMs
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -x > gpurun_out/s3q_tests.log 2>&1; echo tests=$?
tail -1 gpurun_out/s3q_tests.log
cp paper_1604_01879_b200/libgift.so /tmp/libgift_prod.so
for v in 16 8 28; do
if [ $v != 16 ]; then cp tools/libgift_sp_$v.so paper_1604_01879_b200/libgift.so; else cp /tmp/libgift_prod.so paper_1604_01879_b200/libgift.so; fi
for cfg in "1 0" "2 20"; do set -- $cfg
timeout 1200 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline --lanes $1 --reserve-sms $2 > gpurun_out/s3q_c4_$v_l$1.json 2>/dev/null
tail -1 gpurun_out/s3q_c4_$v_l$1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('side $v lanes $1 reserve $2', round(d['value']), round(d['e2e']['value']), round(r['scan_ms_avg'],2), round(d['ms_per_step'],2))"
done
done
cp /tmp/libgift_prod.so paper_1604_01879_b200/libgift.so
