#!/bin/bash
# session-2 measurement set: full GPU suite, every config's bench line, reference arm C2
mkdir -p gpurun_out
export GIFT_PARITY_OUT=gpurun_out/s2x_parity.jsonl
export GIFT_REFSUITE_OUT=gpurun_out/s2x_refsuite.log
rm -f $GIFT_PARITY_OUT
timeout 3000 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/s2x_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/s2x_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/s2x_c2.json 2> gpurun_out/s2x_c2.err; echo c2=$?
timeout 600 python bench.py --config c1 --steps 20 --warmup 5 > gpurun_out/s2x_c1.json 2> gpurun_out/s2x_c1.err; echo c1=$?
timeout 1500 python bench.py --config c3 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/s2x_c3.json 2> gpurun_out/s2x_c3.err; echo c3=$?
timeout 1800 python bench.py --config c4 --steps 8 --warmup 3 > gpurun_out/s2x_c4.json 2> gpurun_out/s2x_c4.err; echo c4=$?
timeout 900 python bench.py --config c5 --steps 10 --warmup 3 > gpurun_out/s2x_c5.json 2> gpurun_out/s2x_c5.err; echo c5=$?
timeout 1500 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/s2x_ref.json 2> gpurun_out/s2x_ref.err; echo ref=$?
for f in c1 c2 c3 c4 c5; do tail -1 gpurun_out/s2x_$f.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline') or {}; print('$f', round(d['value']), round(d['e2e']['value']), r.get('scan_ms_avg'), r.get('frac'), d.get('clocks'))"; done
tail -1 gpurun_out/s2x_ref.json | head -c 300
