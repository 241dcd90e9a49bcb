#!/bin/bash
# relaxed TMEM hand-back arrives: variant tests, traces, C4 and C2 benches
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_variants.py -q -x > gpurun_out/s2m_variants.log 2>&1; echo variants=$?
tail -1 gpurun_out/s2m_variants.log
cp paper_1604_01879_b200/libgift.so /tmp/libgift_prod.so
timeout 600 python tools/scan_trace.py c4s > gpurun_out/s2m_trace_c4s.log 2>&1; echo trace=$?
grep "scan\|median\|tail parts" gpurun_out/s2m_trace_c4s.log | head -4
cp /tmp/libgift_prod.so paper_1604_01879_b200/libgift.so
timeout 1800 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/s2m_c4.json 2> gpurun_out/s2m_c4.err; echo c4=$?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s2m_c2.json 2> gpurun_out/s2m_c2.err; echo c2=$?
for f in c4 c2; do tail -1 gpurun_out/s2m_$f.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$f', d['value'], d['e2e']['value'], r['scan_ms_avg'], r['frac'])"; done
