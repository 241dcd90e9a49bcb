#!/bin/bash
# HEAD check: full GPU suite, smoke, default bench (C2), C4 and C5 lines
mkdir -p gpurun_out
export GIFT_REFSUITE_OUT=gpurun_out/s4s_reference_suite.txt
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s4s_tests.log 2>&1; echo tests=$?
tail -1 gpurun_out/s4s_tests.log
grep -E "^FAILED|^ERROR" gpurun_out/s4s_tests.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4s_smoke.log 2>&1; echo smoke=$?
tail -1 gpurun_out/s4s_smoke.log
for c in c2 c4 c5; do
timeout 1800 python bench.py --config $c > gpurun_out/s4s_$c.json 2> gpurun_out/s4s_$c.err; echo $c=$?
grep "^{" gpurun_out/s4s_$c.json | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline') or {}; print('$c', round(d['value']), round(d['e2e']['value']), d['ms_per_step'], r.get('frac'), d['clocks'])"
done
