#!/bin/bash
# hash S-IF query: parity tests, C5 bench (hash vs bucket), launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sif" > gpurun_out/s3c_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/s3c_tests.log
timeout 1200 python -m pytest tests/test_gpu_config_scale.py -q -x -k c5 > gpurun_out/s3c_c5test.log 2>&1; echo c5test=$?
tail -2 gpurun_out/s3c_c5test.log
for m in hash bucket; do
timeout 900 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline --sif $m > gpurun_out/s3c_c5_$m.json 2> gpurun_out/s3c_c5_$m.err; echo c5_$m=$?
tail -1 gpurun_out/s3c_c5_$m.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$m', d['value'], d['e2e']['value'], r['sif_ms_avg'], r['frac'])"
done
CMD="python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --sif hash"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s3c_launches_c5.csv $CMD > /dev/null 2>&1; echo launches=$?
