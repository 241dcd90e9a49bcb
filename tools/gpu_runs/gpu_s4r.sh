#!/bin/bash
# owner reduce: two segments per thread in the fast kernel; owner/reduce tests, C4 config-scale parity, C4 bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_sharded.py tests/test_gpu_config_scale.py -q -k "owner or reduce or variants or c4 or sharded or dense or many_probes" > gpurun_out/s4r_tests.log 2>&1; echo tests=$?
tail -1 gpurun_out/s4r_tests.log
grep -E "^FAILED" gpurun_out/s4r_tests.log | head
for i in 1 2; do
timeout 1800 python bench.py --config c4 --no-cpu-baseline > gpurun_out/s4r_c4_$i.json 2> gpurun_out/s4r_c4_$i.err
grep "^{" gpurun_out/s4r_c4_$i.json | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d['clocks'])"
done
timeout 1500 python tools/lane_trace.py --config c4 --lanes 1 --steps 8 > gpurun_out/s4r_trace_c4_l1.json 2> /dev/null; tail -1 gpurun_out/s4r_trace_c4_l1.json | cut -c1-700
