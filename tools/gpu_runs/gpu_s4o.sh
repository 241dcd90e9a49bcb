#!/bin/bash
# Session-4 final measurement set (after the S-IF bucket and ranking changes): GPU suite, smoke, every config's bench line, reference arm
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/s4o_gpu.txt
export GIFT_PARITY_OUT=gpurun_out/s4o_parity.jsonl GIFT_REFSUITE_OUT=gpurun_out/s4o_reference_suite.txt
timeout 2400 python -m pytest tests -m gpu -q --durations=40 > gpurun_out/s4o_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/s4o_tests.log
grep -E "^FAILED|^ERROR" gpurun_out/s4o_tests.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4o_smoke.log 2>&1; echo smoke=$?
tail -1 gpurun_out/s4o_smoke.log
timeout 900 python bench.py > gpurun_out/s4o_c2.json 2> gpurun_out/s4o_c2.err; echo c2=$?
for c in c1 c5 c4 c3; do
timeout 1800 python bench.py --config $c > gpurun_out/s4o_$c.json 2> gpurun_out/s4o_$c.err; echo $c=$?
done
for c in c2 c1 c5 c4 c3; do
grep "^{" gpurun_out/s4o_$c.json | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline') or {}; print('$c', round(d['value']), round(d['e2e']['value']), d['ms_per_step'], r.get('frac'), d['clocks'])"
done
timeout 1200 python bench.py --impl reference > gpurun_out/s4o_ref.json 2> gpurun_out/s4o_ref.err; echo ref=$?
tail -1 gpurun_out/s4o_ref.json | cut -c1-300
