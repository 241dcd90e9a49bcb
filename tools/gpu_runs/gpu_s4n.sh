#!/bin/bash
# rank kernel sorts over the occupied power of two: S-IF tests, C5 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_config_scale.py tests/test_gpu_parity.py tests/test_gpu_edges.py -q -k "c5 or sif or rerank or top_k" > gpurun_out/s4n_tests.log 2>&1; echo tests=$?
tail -1 gpurun_out/s4n_tests.log
for i in 1 2; do
timeout 900 python bench.py --config c5 --no-cpu-baseline > gpurun_out/s4n_c5_$i.json 2> gpurun_out/s4n_c5.err; echo c5=$?
grep "^{" gpurun_out/s4n_c5_$i.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', round(d['value']), round(d['e2e']['value']), d['roofline']['sif_ms_avg'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:sif_ --csv --log-file gpurun_out/s4n_launches_c5.csv python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --lanes 1 > /dev/null 2>&1; echo ncu=$?
