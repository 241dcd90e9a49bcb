#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s2y_c5.json 2> gpurun_out/s2y_c5.err; echo c5=$?
tail -1 gpurun_out/s2y_c5.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], json.dumps(d['roofline']))"
tail -3 gpurun_out/s2y_c5.err
