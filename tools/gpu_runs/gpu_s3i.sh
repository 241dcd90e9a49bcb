#!/bin/bash
# owner reduce split: single-segment shapes on fif_owner_fast_kernel
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_sharded.py tests/test_gpu_streamed.py -q -x > gpurun_out/s3i_tests.log 2>&1; echo tests=$?
tail -1 gpurun_out/s3i_tests.log
timeout 1200 python -m pytest tests/test_gpu_config_scale.py -q -x -k "c4 or c3" > gpurun_out/s3i_scale.log 2>&1; echo scale=$?
tail -1 gpurun_out/s3i_scale.log
CMD="python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --lanes 1 --reserve-sms 0"
timeout 1500 ncu --nvtx --nvtx-include "gift.query_batch/" -k regex:owner --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3i_own.csv $CMD > /dev/null 2>&1; echo own=$?
python tools/launch_table.py gpurun_out/s3i_own.csv | sed -n 2,3p
for cfg in "1 0" "2 20" "2 8"; do set -- $cfg
timeout 1200 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline --lanes $1 --reserve-sms $2 > gpurun_out/s3i_c4_l$1_r$2.json 2>/dev/null
tail -1 gpurun_out/s3i_c4_l$1_r$2.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c4 lanes $1 reserve $2', round(d['value']), round(d['e2e']['value']), round(r['scan_ms_avg'],2), round(d['ms_per_step'],2))"
done
