#!/bin/bash
# dense-cell probe-major scan: variant tests, fp16 parity, c4s trace, C4 bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_variants.py -q -x > gpurun_out/s2i_variants.log 2>&1; echo variants=$?
tail -15 gpurun_out/s2i_variants.log | grep -v "^$" | tail -8
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fp16" > gpurun_out/s2i_parity.log 2>&1; echo parity=$?
tail -2 gpurun_out/s2i_parity.log
cp paper_1604_01879_b200/libgift.so /tmp/libgift_prod.so
timeout 600 python tools/scan_trace.py c4s > gpurun_out/s2i_trace_c4s.log 2>&1; echo trace=$?
grep "scan\|median" gpurun_out/s2i_trace_c4s.log | head -6
cp /tmp/libgift_prod.so paper_1604_01879_b200/libgift.so
timeout 1800 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/s2i_c4.json 2> gpurun_out/s2i_c4.err; echo c4=$?
tail -1 gpurun_out/s2i_c4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c4', d['value'], d['e2e']['value'], r['scan_ms_avg'], r['frac'])"
