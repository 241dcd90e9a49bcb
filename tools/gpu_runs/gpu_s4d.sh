#!/bin/bash
# C1 with CUDA-graph lanes: tests, lanes sweep graph on/off
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "query_many or graphed" > gpurun_out/s4d_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/s4d_tests.log
for g in off on; do for L in 1 2 4 6; do
timeout 600 python bench.py --config c1 --steps 20 --warmup 5 --no-cpu-baseline --graph $g --lanes $L > gpurun_out/s4d_c1_${g}_$L.json 2> gpurun_out/s4d_c1_${g}_$L.err
tail -1 gpurun_out/s4d_c1_${g}_$L.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('graph $g lanes $L', round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4))" || tail -3 gpurun_out/s4d_c1_${g}_$L.err
done; done
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --graph on > gpurun_out/s4d_c2_on.json 2> gpurun_out/s4d_c2_on.err
tail -1 gpurun_out/s4d_c2_on.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2 graph on', round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4))" || tail -3 gpurun_out/s4d_c2_on.err
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s4d_c2_off.json 2> gpurun_out/s4d_c2_off.err
tail -1 gpurun_out/s4d_c2_off.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2 graph off', round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4))" || tail -3 gpurun_out/s4d_c2_off.err
