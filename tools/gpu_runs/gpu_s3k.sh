#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --config c5 --steps 12 --warmup 3 > gpurun_out/s3k_c5.json 2> gpurun_out/s3k_c5.err; echo c5=$?
tail -1 gpurun_out/s3k_c5.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d['run']['lanes'], d['cpu_baseline']['value'])"
timeout 600 python -m pytest tests/test_bench_contract.py -q 2>&1 | tail -1
