#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_variants.py -q -x > gpurun_out/s2q_variants.log 2>&1; echo variants=$?
tail -1 gpurun_out/s2q_variants.log
cp paper_1604_01879_b200/libgift.so /tmp/libgift_prod.so
timeout 600 python tools/scan_trace.py c4s 0 0 1 > gpurun_out/s2q_trace_dense.log 2>&1; echo trace=$?
grep "scan\|median\|parts" gpurun_out/s2q_trace_dense.log | head -5
cp /tmp/libgift_prod.so paper_1604_01879_b200/libgift.so
timeout 1800 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/s2q_c4.json 2> gpurun_out/s2q_c4.err; echo c4=$?
tail -1 gpurun_out/s2q_c4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c4', d['value'], d['e2e']['value'], r['scan_ms_avg'], r['frac'])"
