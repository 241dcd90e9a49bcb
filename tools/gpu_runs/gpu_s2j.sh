#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_variants.py -q -x -k "dense or fp16" > gpurun_out/s2j_variants.log 2>&1; echo variants=$?
tail -2 gpurun_out/s2j_variants.log
cp paper_1604_01879_b200/libgift.so /tmp/libgift_prod.so
timeout 600 python tools/scan_trace.py c4s > gpurun_out/s2j_trace_c4s.log 2>&1; echo trace=$?
grep "scan\|median" gpurun_out/s2j_trace_c4s.log | head -6
timeout 600 python tools/scan_trace.py c4s 8 > gpurun_out/s2j_trace_c4s_d8.log 2>&1; echo trace=$?
grep "scan\|median" gpurun_out/s2j_trace_c4s_d8.log | head -6
cp /tmp/libgift_prod.so paper_1604_01879_b200/libgift.so
timeout 1800 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/s2j_c4.json 2> gpurun_out/s2j_c4.err; echo c4=$?
tail -1 gpurun_out/s2j_c4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c4', d['value'], d['e2e']['value'], r['scan_ms_avg'], r['frac'])"
