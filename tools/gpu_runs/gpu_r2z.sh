#!/bin/bash
# bucketed S-IF query: parity, C5 bench (bucket vs sort), launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sparse_sif or bucketed" > gpurun_out/r2zg_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/r2zg_tests.log
timeout 1200 python -m pytest tests/test_gpu_config_scale.py -q -x -k c5 > gpurun_out/r2zg_c5test.log 2>&1; echo c5test=$?
tail -3 gpurun_out/r2zg_c5test.log
for m in bucket sort; do
  timeout 600 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline --sif $m > gpurun_out/r2zg_c5_$m.json 2> gpurun_out/r2zg_c5_$m.err; echo bench_$m=$?
  tail -1 gpurun_out/r2zg_c5_$m.json | head -c 400; echo
done
CMD="python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --sif bucket"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2zg_launches_c5.csv $CMD > gpurun_out/r2zg_ncu.log 2>&1; echo launches=$?
