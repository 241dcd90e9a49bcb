#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "owner or reduce or e2e" > gpurun_out/s3h_tests.log 2>&1; echo tests=$?
tail -1 gpurun_out/s3h_tests.log
CMD="python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --lanes 1 --reserve-sms 0"
timeout 1500 ncu --nvtx --nvtx-include "gift.query_batch/" -k regex:owner_reduce --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3h_own.csv $CMD > /dev/null 2>&1; echo own=$?
python tools/launch_table.py gpurun_out/s3h_own.csv | sed -n 2p
