#!/bin/bash
# shuffle-reduce tail: scan parity tests, c4s trace, C4/C2 benches
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/s2c_parity.log 2>&1; echo parity=$?
tail -3 gpurun_out/s2c_parity.log
cp paper_1604_01879_b200/libgift.so /tmp/libgift_prod.so
timeout 600 python tools/scan_trace.py c4s > gpurun_out/s2c_trace_c4s.log 2>&1; echo trace=$?
cp /tmp/libgift_prod.so paper_1604_01879_b200/libgift.so
timeout 1800 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/s2c_c4.json 2> gpurun_out/s2c_c4.err; echo c4=$?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s2c_c2.json 2> gpurun_out/s2c_c2.err; echo c2=$?
for f in c4 c2; do tail -1 gpurun_out/s2c_$f.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$f', d['value'], d['e2e']['value'], r['scan_ms_avg'], r['frac'])"; done
