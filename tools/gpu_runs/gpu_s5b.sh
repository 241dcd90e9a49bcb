#!/bin/bash
# session 5: S-IF tests + C5 bench after the sort-path bound cap; C3 bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config_scale.py tests/test_gpu_variants.py -m gpu -q > gpurun_out/s5b_tests.log 2>&1; echo tests=$?
tail -1 gpurun_out/s5b_tests.log
grep -E "^FAILED|^ERROR" gpurun_out/s5b_tests.log | head
for c in c5 c3; do
timeout 600 python bench.py --config $c > gpurun_out/s5b_$c.json 2> gpurun_out/s5b_$c.err; echo $c=$?
grep "^{" gpurun_out/s5b_$c.json | tail -1 | cut -c1-260
done
