#!/bin/bash
# owner reduce: single-segment shapes skip the shape lookups
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_sharded.py tests/test_gpu_streamed.py -q -x > gpurun_out/s2v_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/s2v_tests.log
timeout 1200 python -m pytest tests/test_gpu_config_scale.py -q -x -k "c4 or c3" > gpurun_out/s2v_scale.log 2>&1; echo scale=$?
tail -2 gpurun_out/s2v_scale.log
timeout 1800 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/s2v_c4.json 2> gpurun_out/s2v_c4.err; echo c4=$?
tail -1 gpurun_out/s2v_c4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c4', d['value'], d['e2e']['value'], r['scan_ms_avg'], r['frac'], d['ms_per_step'])"
CMD="python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --lanes 1 --reserve-sms 0"
timeout 1500 ncu --nvtx --nvtx-include "gift.query_batch/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s2v_launches_c4.csv $CMD > gpurun_out/s2v_ncu1.log 2>&1; echo launches=$?
